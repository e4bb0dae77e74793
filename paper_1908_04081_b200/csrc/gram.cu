// gram.cu -- K_gram: G = Y^T Y of the tall-skinny fp64 basis, single pass.
//
// Reference: lacore.py:37-47 `gram` (OpenBLAS dgemm `y.T @ y`, lower triangle
// mirrored so G is exactly symmetric).
//
// Y (n x k, k = 2 s + 1 <= 33, column-major, ld a multiple of GT_ROWS with the
// padding rows zeroed at allocation) streams through shared memory in
// GT_ROWS-row tiles with a GT_STAGES-deep TMA pipeline (one 1 KB cp.async.bulk
// per column per tile, mbarrier completion, issued by one thread); each warp feeds
// 4-row slices of the tile to the fp64 tensor core (DMMA, mma.m8n8k4.f64): with
// the column blocks Y_i (8 columns) the warp accumulates the lower-triangular
// tiles G_ij += Y_i^T Y_j.  The A and B fragments of m8n8k4 have the same
// layout for a Gram product (thread (g, t) holds Y[row0 + t, 8 i + g]), so one
// fragment load per column block serves every tile in its row and column.
// Per-warp accumulators are combined in a fixed warp order, per-CTA partials
// are written packed, and the last CTA to finish sums them in CTA order:
// deterministic, one launch, no atomics on data.
//
// Roofline: HBM-bound (8 k bytes/row against k(k+1)/2 FMA/row).
#include "internal.cuh"

namespace {

#ifndef GT_ROWS_DEF
#define GT_ROWS_DEF 128
#endif
#ifndef GT_STAGES_DEF
#define GT_STAGES_DEF 4
#endif
constexpr int GT_ROWS = GT_ROWS_DEF;
constexpr int GT_STAGES = GT_STAGES_DEF;
constexpr int GT_LD = GT_ROWS + 4;  // LD % 16 == 4: conflict-free fragment loads
constexpr int GT_CONSUMERS = 8;                    // DMMA warps (16 rows of a tile each)
constexpr int GT_THREADS = (GT_CONSUMERS + 1) * 32;  // + one TMA producer warp

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0, spins = 0;
  while (!done) {
    if (++spins > (1u << 26)) __trap();
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// NB full 8-column blocks go through DMMA; the REM (<= 2) trailing columns are
// accumulated on the CUDA cores (padding them to a 9th..16th column would double
// the tensor work and make the kernel DMMA-bound instead of HBM-bound).
// PACKED=false: `out` = full symmetric k x k matrix (unit entry point).
// PACKED=true:  `out` = [packed lower triangle | sum(norm_t) | sum(norm_r)], the
//               one buffer an outer loop allreduces (norm_* = level-0 partials).
template <int NB, int REM, bool PACKED>
__device__ __forceinline__ void gram_body(const double* __restrict__ Y, int64_t ld, int64_t nrows,
                                          int k, double* part, double* out, int* counter,
                                          const double* norm_t, const double* norm_r, int n_norm) {
  constexpr int T = NB * (NB + 1) / 2;
  constexpr int NC = NB * 8 + REM;  // columns staged per tile
  extern __shared__ __align__(16) double gsm[];
  double* tiles = gsm;                              // [GT_STAGES][NC][GT_LD]
  double* red = gsm + GT_STAGES * NC * GT_LD;       // [T][64] + [REM][NB*8 + REM]
  double* redr = red + T * 64;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int64_t ntiles = (nrows + GT_ROWS - 1) / GT_ROWS;  // rows >= nrows read as 0

  // zero the padding columns (k .. NC-1) of every stage once
  for (int i = tid; i < GT_STAGES * NC * GT_LD; i += GT_THREADS) {
    int cc = (i / GT_LD) % NC;
    if (cc >= k) tiles[i] = 0.0;
  }
  double acc[T > 0 ? T : 1][2];
#pragma unroll
  for (int q = 0; q < T; ++q) acc[q][0] = acc[q][1] = 0.0;
  double accr[REM > 0 ? REM : 1][NB + 1];  // remainder column x (block cb column g) / x rem
#pragma unroll
  for (int a = 0; a < (REM > 0 ? REM : 1); ++a)
#pragma unroll
    for (int cb = 0; cb <= NB; ++cb) accr[a][cb] = 0.0;

  const int kc = k < NC ? k : NC;
  // warp-specialised pipeline: warp GT_CONSUMERS produces (TMA bulk copies into
  // stage s after `empty[s]` completes), warps 0..7 consume (wait `full[s]`,
  // DMMA, arrive on `empty[s]`) -- no CTA-wide barrier per tile
  __shared__ __align__(8) uint64_t full[GT_STAGES], empty[GT_STAGES];
  if (tid == 0) {
    for (int st = 0; st < GT_STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], GT_CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == GT_CONSUMERS) {
    if (lane == 0) {
      int64_t kk = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++kk) {
        const int stage = (int)(kk % GT_STAGES);
        if (kk >= GT_STAGES) mbar_wait(&empty[stage], (uint32_t)(((kk / GT_STAGES) - 1) & 1));
        double* dst = tiles + (size_t)stage * NC * GT_LD;
        const double* src = Y + tile * GT_ROWS;
        mbar_arrive_tx(&full[stage], (uint32_t)(kc * GT_ROWS * sizeof(double)));
        for (int cc = 0; cc < kc; ++cc)
          bulk_g2s(dst + cc * GT_LD, src + (int64_t)cc * ld, GT_ROWS * sizeof(double), &full[stage]);
      }
    }
  } else {
    int64_t kk = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++kk) {
      const int stage = (int)(kk % GT_STAGES);
      mbar_wait(&full[stage], (uint32_t)((kk / GT_STAGES) & 1));
      const double* ts = tiles + (size_t)stage * NC * GT_LD;
      const int64_t valid = nrows - tile * GT_ROWS;  // rows of this tile below nrows
      // 8 warps x 16 rows = 128 rows: four k-steps of 4 rows per warp
#pragma unroll
      for (int ks = 0; ks < GT_ROWS / 32; ++ks) {
        const int row0 = warp * (GT_ROWS / 8) + ks * 4;
        const bool live = row0 + t4 < valid;
        double fr[NB > 0 ? NB : 1];
#pragma unroll
        for (int cb = 0; cb < NB; ++cb) fr[cb] = live ? ts[(cb * 8 + g) * GT_LD + row0 + t4] : 0.0;
        int q = 0;
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j, ++q) dmma(acc[q][0], acc[q][1], fr[i], fr[j]);
        if (REM > 0) {
#pragma unroll
          for (int a = 0; a < REM; ++a) {
            const double yr = live ? ts[(NB * 8 + a) * GT_LD + row0 + t4] : 0.0;
#pragma unroll
            for (int cb = 0; cb < NB; ++cb) accr[a][cb] = fma(yr, fr[cb], accr[a][cb]);
            // remainder x remainder (columns NB*8 .. NB*8+a), lanes g <= a
            if (g <= a) {
              const double yb = live ? ts[(NB * 8 + g) * GT_LD + row0 + t4] : 0.0;
              accr[a][NB] = fma(yr, yb, accr[a][NB]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);  // this warp is done with the stage
    }
  }
  __syncthreads();

  // remainder partials: sum over the 4 row lanes (t4) of each g
  if (REM > 0) {
#pragma unroll
    for (int a = 0; a < REM; ++a)
#pragma unroll
      for (int cb = 0; cb <= NB; ++cb) {
        double v = accr[a][cb];
        v += __shfl_down_sync(0xffffffffu, v, 2);
        v += __shfl_down_sync(0xffffffffu, v, 1);
        accr[a][cb] = v;  // valid in lanes with t4 == 0
      }
  }
  // combine warps in fixed order: red[q][g*8 + 2 t4 + e], redr[a][col]
  for (int w = 0; w < GT_CONSUMERS; ++w) {
    if (warp == w) {
#pragma unroll
      for (int q = 0; q < T; ++q) {
        double* d = red + q * 64 + g * 8 + 2 * t4;
        if (w == 0) {
          d[0] = acc[q][0];
          d[1] = acc[q][1];
        } else {
          d[0] += acc[q][0];
          d[1] += acc[q][1];
        }
      }
      if (REM > 0 && t4 == 0) {
#pragma unroll
        for (int a = 0; a < REM; ++a) {
#pragma unroll
          for (int cb = 0; cb < NB; ++cb) {
            double* d = redr + a * NC + cb * 8 + g;
            *d = (w == 0) ? accr[a][cb] : *d + accr[a][cb];
          }
          if (g <= a) {
            double* d = redr + a * NC + NB * 8 + g;
            *d = (w == 0) ? accr[a][NB] : *d + accr[a][NB];
          }
        }
      }
    }
    __syncthreads();
  }
  // packed lower triangle of this CTA
  const int npack = k * (k + 1) / 2;
  for (int e = tid; e < npack; e += GT_THREADS) {
    int a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while (a * (a + 1) / 2 > e) --a;
    while ((a + 1) * (a + 2) / 2 <= e) ++a;
    const int b = e - a * (a + 1) / 2;
    double v;
    if (a >= NB * 8) {  // remainder row a, column b <= a
      v = redr[(a - NB * 8) * NC + b];
    } else {
      const int bi = a >> 3, bj = b >> 3;
      const int q = bi * (bi + 1) / 2 + bj;
      v = red[q * 64 + (a & 7) * 8 + (b & 7)];
    }
    part[(size_t)blockIdx.x * GPACK + e] = v;
  }
  // last CTA: fixed-order sum over CTAs, mirror to a full symmetric matrix
  __threadfence();
  __shared__ int ticket;
  __syncthreads();
  if (tid == 0) ticket = atomicAdd(counter, 1);
  __syncthreads();
  if (ticket != (int)gridDim.x - 1) return;
  __threadfence();
  const int nb = gridDim.x;
  for (int e = tid; e < npack; e += GT_THREADS) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int cta = 0;
    const volatile double* pp = part + e;
    for (; cta + 4 <= nb; cta += 4) {
      s0 += pp[(size_t)(cta + 0) * GPACK];
      s1 += pp[(size_t)(cta + 1) * GPACK];
      s2 += pp[(size_t)(cta + 2) * GPACK];
      s3 += pp[(size_t)(cta + 3) * GPACK];
    }
    for (; cta < nb; ++cta) s0 += pp[(size_t)cta * GPACK];
    const double v = (s0 + s1) + (s2 + s3);
    if (PACKED) {
      out[e] = v;
    } else {
      int a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (a * (a + 1) / 2 > e) --a;
      while ((a + 1) * (a + 2) / 2 <= e) ++a;
      const int b = e - a * (a + 1) / 2;
      out[a * k + b] = v;
      out[b * k + a] = v;
    }
  }
  if (PACKED && warp == 0) {  // level-0 residual norms, fixed-order tree
    double st = 0.0, sr = 0.0;
    for (int i = lane; i < n_norm; i += 32) {
      st += norm_t[i];
      sr += norm_r[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      st += __shfl_down_sync(0xffffffffu, st, o);
      sr += __shfl_down_sync(0xffffffffu, sr, o);
    }
    if (lane == 0) {
      out[npack] = st;
      out[npack + 1] = sr;
    }
  }
  if (tid == 0) *counter = 0;
}

template <int NB, int REM>
__global__ void __launch_bounds__(GT_THREADS) k_gram_state(Ctx c) {
  if (c.st->done) return;
  TL_K(c, 0);
  TL_BEGIN(c, 16);
  gram_body<NB, REM, true>(c.Y, c.ld, c.n_own, c.cfg->ncols, c.part_g, c.red_buf,
                           &c.st->gram_count, c.part_t, c.part_r, c.red_n);
  TL_END(c, 16);
}

template <int NB, int REM>
__global__ void __launch_bounds__(GT_THREADS)
    k_gram_raw(const double* Y, int64_t ld, int64_t n, int k, double* part, double* out,
               int* counter) {
  gram_body<NB, REM, false>(Y, ld, n, k, part, out, counter, nullptr, nullptr, 0);
}

template <int NB, int REM>
constexpr size_t gram_smem() {
  return sizeof(double) * ((size_t)GT_STAGES * (NB * 8 + REM) * GT_LD +
                           (size_t)(NB * (NB + 1) / 2) * 64 + (size_t)REM * (NB * 8 + REM) + 8);
}

template <int NB, int REM>
void set_attr() {
  static std::atomic<unsigned long long> done{0};  // per device
  if (first_use_on_device(done)) {
    cudaFuncSetAttribute(k_gram_state<NB, REM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)gram_smem<NB, REM>());
    cudaFuncSetAttribute(k_gram_raw<NB, REM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)gram_smem<NB, REM>());
    mark_device_done(done);
  }
}

int gram_grid(int64_t rows) {
  int64_t t = (rows + GT_ROWS - 1) / GT_ROWS;
  if (t > 2 * NUM_SMS) t = 2 * NUM_SMS;  // 2 CTAs per SM (shared-memory bound)
  return (int)(t < 1 ? 1 : t);
}

}  // namespace

int gram_row_multiple() { return GT_ROWS; }

// k columns -> NB DMMA blocks + REM CUDA-core columns (REM = k mod 8 when <= 2,
// otherwise the last block is zero-padded for DMMA)
#define GRAM_DISPATCH(K, LAUNCH)                                      \
  do {                                                                \
    const int nb_ = (K) / 8, r_ = (K) % 8;                            \
    switch (r_ <= 2 ? nb_ * 10 + r_ : (nb_ + 1) * 10) {               \
      case 1: LAUNCH(0, 1); break;                                    \
      case 2: LAUNCH(0, 2); break;                                    \
      case 10: LAUNCH(1, 0); break;                                   \
      case 11: LAUNCH(1, 1); break;                                   \
      case 12: LAUNCH(1, 2); break;                                   \
      case 20: LAUNCH(2, 0); break;                                   \
      case 21: LAUNCH(2, 1); break;                                   \
      case 22: LAUNCH(2, 2); break;                                   \
      case 30: LAUNCH(3, 0); break;                                   \
      case 31: LAUNCH(3, 1); break;                                   \
      case 32: LAUNCH(3, 2); break;                                   \
      case 40: LAUNCH(4, 0); break;                                   \
      case 41: LAUNCH(4, 1); break;                                   \
      case 42: LAUNCH(4, 2); break;                                   \
      case 50: LAUNCH(5, 0); break;                                   \
      default: break;                                                 \
    }                                                                 \
  } while (0)

void launch_gram(const Ctx& c, int ncols, cudaStream_t s) {
  const int grid = gram_grid(c.n_own);
#define L_STATE(NB, REM)                                                          \
  set_attr<NB, REM>();                                                            \
  k_gram_state<NB, REM><<<grid, GT_THREADS, gram_smem<NB, REM>(), s>>>(c)
  GRAM_DISPATCH(ncols, L_STATE);
#undef L_STATE
}

void launch_gram_raw(const double* Y, int64_t n, int64_t ld, int k, double* part, double* out,
                     int* counter, cudaStream_t s) {
  const int grid = gram_grid(n);
#define L_RAW(NB, REM)                                                            \
  set_attr<NB, REM>();                                                            \
  k_gram_raw<NB, REM><<<grid, GT_THREADS, gram_smem<NB, REM>(), s>>>(Y, ld, n, k, part, out, counter)
  GRAM_DISPATCH(k, L_RAW);
#undef L_RAW
}
