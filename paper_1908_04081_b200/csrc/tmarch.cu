// tmarch.cu -- K_mpk for 7-point stencil operators: the plane march fed by TMA.
//
// Reference: basis.py:210-225 `_recurrence_columns` over lacore.py:25-34 `spmv`
// (scipy csr_matvec), the same per-row arithmetic as every other level kernel
// (mpk.cu): row sum over the union [-S, -o, -1, 0, +1, +o, +S] in stored order
// with separately rounded products and adds, then the recurrence op by op --
// bit-identical to csr_matvec / the CSR kernels.
//
// Layout: a work item is a 32 x 8 tile of a plane (32 columns of a line, 8
// lines of stride o) marched over zc planes.  Warp 8 of the CTA (one elected
// thread) is the producer: for every plane of its items it issues one 4-D TMA
// box per input vector -- the tile plus its halo, 36 x 10 doubles, out
// of bounds filled with zeros -- plus the tile's 1-byte row ids (and b on level
// 0) into a ring of TM_R shared-memory stages, each completed on an mbarrier
// (expect_tx).  Warps 0-7 are consumers: warp w owns line w of the tile and
// walks the planes keeping x[r - S], x[r], x[r + S] in registers (one
// shared-memory read per vector and plane brings the plane ahead), reading the
// +-1 / +-o neighbours from the staged plane.  Each consumer thread releases a
// stage by its own arrive on the stage's `empty` barrier (256 per phase); there is no
// CTA-wide barrier on the per-plane path, so warps drift by up to the ring
// depth and the producer keeps TM_R - 2 planes of every input vector in flight
// per CTA (the HBM stream the register march could not keep deep enough).
//
// Roofline (HBM): per level 1 byte of row id + 16 bytes per row and generated
// column (in + out; + 8 for a Chebyshev two-back read; + x and b on level 0).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <type_traits>

#include "internal.cuh"
#include "rowops.cuh"

namespace {

// staged tile + halo (doubles): 8 lines + 1 above and below; 32 columns + 2
// each side -- a box's first x coordinate must be 16-byte aligned, so the
// one-cell halo in x is loaded as two (x0 - 2 .. x0 + 33)
constexpr int TM_W = 36, TM_H = 10, TM_XH = 2;
constexpr int TM_BOX = TM_W * TM_H;                // 360
constexpr int TM_BOXB = (TM_BOX * 8 + 127) / 128 * 128;  // 2944: 128-byte aligned boxes
constexpr int TM_THREADS = 288;                    // 8 consumer warps + 1 producer warp
#ifndef TM_MINB
#define TM_MINB 3  // CTAs per SM the register budget must allow (72 registers)
#endif
#ifndef TM_R0
#define TM_R0 TM_R  // ring depth of level 0 (larger stages: x, P_0, R_0, b)
#endif
template <bool L0>
struct Ring {
  static constexpr int R = L0 ? TM_R0 : TM_R;
};

// a stage: the input boxes, then 2 KB tiles without halo -- level 0: b; levels
// >= 1: the two two-back vectors (loaded only when mu != 0) -- then the row ids
__host__ __device__ constexpr int tm_stage_bytes(int nv, bool l0) {
  return nv * TM_BOXB + (l0 ? 2048 : 4096) + 256;
}
__host__ __device__ constexpr uint32_t tm_tx_bytes(int nv, bool l0, bool mu) {
  return (uint32_t)(nv * TM_BOX * 8 + (l0 ? 2048 : mu ? nv * 2048 : 0) + 256);
}
__host__ __device__ inline size_t tm_head_bytes(int pat_np, int zm_np, bool table) {
  // pattern values, then (plane-table plans) each plane's first local row and its plane index
  const size_t a = (size_t)pat_np * SS_MAX_NE * 8 + (table ? 8 * (size_t)zm_np : 0);
  return (a + 127) / 128 * 128;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, int c0, int c1, int c2,
                                            int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];\n" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// consumer wait on a full barrier (phase parity ph): a lost transaction traps
__device__ __forceinline__ void tm_wait(uint32_t bar, uint32_t ph) {
  uint32_t done = 0, spins = 0;
  for (;;) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(ph)
        : "memory");
    if (done) break;
    if (++spins > (1u << 26)) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive_plain(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumers_bar() {
  asm volatile("bar.sync 1, 256;\n" ::: "memory");
}

template <bool UNIT>
__device__ __forceinline__ double tm_recur(double ay, double y, double y2, double th, double ga,
                                           double mu, bool use_mu) {
  double w = __dsub_rn(ay, __dmul_rn(th, y));
  if (use_mu) w = __dsub_rn(w, __dmul_rn(mu, y2));
  return UNIT ? w : __ddiv_rn(w, ga);
}

// One launch of a level.  NV input vectors: level 0 (L0) x, P_0, R_0 -> P_1,
// R_1 (+ ||b - A x||^2 and ||r||^2 partials); levels >= 1 P_l, R_l ->
// P_{l+1}, R_{l+1} (NV = 2) or P alone (NV = 1, the block's last level).  RK:
// bit 0 non-unit gamma, bit 1 two-back term (mu != 0) -- read from the device
// state, so the kernel picks the instantiation (the graph is captured once).
// dyn: levels >= 1 claim items from a counter while a Leja chain runs beside
// them (a CTA whose SM slot a Leja kernel holds starts late and takes fewer
// items); level 0 keeps a fixed assignment (deterministic norm partials).
struct TmShared {
  uint64_t* full;
  uint64_t* empty;
  int* sitem;
  int* sbase;  // with sitem: the largest plane base of the item's planes (plane-table plans)
  double (*red)[8];
  const double* pval;
  const int* ptab;
  unsigned char* stg;
};

// work item -> (tile, planes [z0, z1))
template <bool L0>
__device__ __forceinline__ void tm_item(const Ctx& c, int it, int ncb, int& cb, int& z0, int& z1) {
  const int zcs = L0 ? c.zm_zc0 : c.zm_zc;
  cb = it % ncb;
  z0 = (it / ncb) * zcs;
  z1 = min(z0 + zcs, c.zm_np);
}

template <int NV, bool L0, int RK, bool EX>
__device__ __forceinline__ void tm_body(const Ctx& c, int l, const ZmPtrs& zp, const TmMaps& maps,
                                        const TmShared& sh, bool dyn, bool do_r) {
  constexpr bool UNIT = (RK & 1) == 0, MU = (RK & 2) != 0 && !L0;
  constexpr int RING = Ring<L0>::R;
  constexpr int NO = L0 ? NV - 1 : NV;  // output vectors
  constexpr int Q0 = L0 ? 1 : 0;        // first input with an output
  constexpr int SB = tm_stage_bytes(L0 ? 3 : 2, L0);  // stage stride (the kernel's largest NV)
  constexpr int IDO = (L0 ? 3 : 2) * TM_BOXB + (L0 ? 2048 : 4096);  // row ids within a stage
  constexpr int YMO = 2 * TM_BOXB;  // two-back tiles within a stage (levels >= 1)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool table = c.zm_base != nullptr;
  const int S = (int)c.zm_S, o = c.zm_o, lines = S / o, ntx = o >> 5;
  const int ncb = ntx * ((lines + 7) >> 3);
  const int np = c.zm_np;
  const int items = (int)(L0 ? c.zm_items0 : c.zm_items);
  const int sigma = c.cfg->sigma;
  uint64_t* full = sh.full;
  uint64_t* empty = sh.empty;
  unsigned char* stg = sh.stg;

  if (warp == 8) {  // ---------------------------------------------- producer
    if (lane != 0) return;
    // Y columns of the inputs (4-D map [col][plane][line][x]); level 0's x has
    // its own 3-D map
    int colq[3];
    if (L0) {
      colq[0] = -1;
      colq[1] = 0;
      colq[2] = sigma + 1;
    } else {
      colq[0] = l;
      colq[1] = sigma + 1 + l;
      colq[2] = -1;
    }
    unsigned* ctr = dyn ? c.zm_ctr + 2 * l : nullptr;
    uint32_t k = 0;
    int it = dyn ? (int)atomicAdd(ctr, 1u) : blockIdx.x;
    for (;;) {
      if (it >= items) {  // end marker: one stage carrying item -1, no data
        const int s0 = k % RING;
        if (k >= RING) mbar_wait(&empty[s0], ((k / RING) - 1) & 1);
        sh.sitem[s0] = -1;
        mbar_arrive_plain(&full[s0]);
        break;
      }
      int cb, z0, z1;
      tm_item<L0>(c, it, ncb, cb, z0, z1);
      const int x0 = (cb % ntx) * 32, y0 = (cb / ntx) * 8;
      for (int zz = z0 - 1; zz <= z1; ++zz, ++k) {
        const int s = k % RING;
        if (k >= RING) mbar_wait(&empty[s], ((k / RING) - 1) & 1);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        if (zz == z0 - 1) {
          sh.sitem[s] = it;
          if (table) {  // one thread looks the item's planes up for all 256 consumers
            int mb = 0;
            for (int z = z0; z < z1; ++z) mb = max(mb, sh.ptab[z]);
            sh.sbase[s] = mb;
          }
        }
        // plane coordinate: geometric plane -> local block (plane table) or
        // itself; outside the walk -1 (zero fill)
        const int pz = (zz >= 0 && zz < np) ? (table ? sh.ptab[np + zz] : zz) : -1;
        SSCG_CHECK(pz >= -1 && pz < np + (table ? 64 : 1));
        unsigned char* dst = stg + (size_t)s * SB;
        mbar_arrive_tx(&full[s], tm_tx_bytes(NV, L0, MU));
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          if (L0 && q == 0)
            tma_load_3d(dst, &maps.x, x0 - TM_XH, y0 - 1, pz, &full[s]);
          else
            tma_load_4d(dst + q * TM_BOXB, &maps.y, x0 - TM_XH, y0 - 1, pz, colq[q], &full[s]);
        }
        if (L0) tma_load_3d(dst + 3 * TM_BOXB, &maps.b, x0, y0, pz, &full[s]);
        if (MU) {  // y_{l-1} of the tile (basis.py:217-218), no halo
#pragma unroll
          for (int q = 0; q < NV; ++q)
            tma_load_4d(dst + YMO + q * 2048, &maps.y8, x0, y0, pz, colq[q] - 1, &full[s]);
        }
        tma_load_3d(dst + IDO, &maps.id, x0, y0, pz, &full[s]);
      }
      it = dyn ? (int)atomicAdd(ctr, 1u) : it + (int)gridDim.x;
    }
    if (dyn && atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
      atomicExch(ctr, 0u);  // the last producer out resets the counters for the next launch
      atomicExch(ctr + 1, 0u);
    }
    return;
  }

  // ------------------------------------------------------------- consumers
  // shared-memory addresses as 32-bit shared-window offsets, formed once
  // (every per-plane access below is an explicit ld.shared / mbarrier op)
  const SolverState* st = c.st;
  const double th = st->prm.th[L0 ? 0 : l], ga = st->prm.ga[L0 ? 0 : l];
  const double mu = L0 ? 0.0 : st->prm.mu[l - 1];
  const int plim = (int)lvl_p_rows(c, sigma, L0 ? 0 : l);
  const int rlim = do_r ? (int)lvl_r_rows(c, sigma, L0 ? 0 : l) : 0;
  const int n_own = (int)c.n_own;
  const uint32_t full0 = smem_u32(full), empty0 = smem_u32(empty);
  const uint32_t cpos8 = 8u * (uint32_t)((warp + 1) * TM_W + (lane + TM_XH));
  const uint32_t my0 = smem_u32(stg) + cpos8;                       // centre, stage 0, vector 0
  const uint32_t id0 = smem_u32(stg) + IDO + (uint32_t)(warp * 32 + lane);  // row id, stage 0
  const uint32_t pv0 = smem_u32(sh.pval);
  const uint32_t b0 = smem_u32(stg) + 3 * TM_BOXB + 8u * (uint32_t)(warp * 32 + lane);  // level 0's b
  const uint32_t ym0 = smem_u32(stg) + YMO + 8u * (uint32_t)(warp * 32 + lane);  // two-back, vector 0
  double tt = 0.0, rr = 0.0;
  unsigned badm = 0;
  int s = 0;        // stage of the next plane to consume
  uint32_t ph = 0;  // its phase parity
  auto advance = [&]() {
    if (++s == RING) {
      s = 0;
      ph ^= 1u;
    }
  };
  // one plane of the walk: wait for plane z + 1 (its centre -> nn), row z
  // from the current stage sc with x[r - S] = p, x[r] = c, x[r + S] = nn;
  // then release sc.  Every consumer thread arrives on `empty` itself (256
  // arrivals per phase: no warp-level sync on the per-plane path).  CHECK:
  // the item may hold rows outside this level's range (tile past the last
  // line, ghost depth beyond the level) -- else every row computes.
  // rb: first local row of plane z, carried from step to step -- the plane
  // table (partitioned plans) is read one plane ahead, beside the row's work,
  // not between the stage wait and the first store address
  int rb = 0;
  auto step = [&](auto check, double (&p)[NV], double (&cc)[NV], double (&nn)[NV], int z,
                  int rel, int& sc) {
    constexpr bool CHECK = decltype(check)::value;
    tm_wait(full0 + 8u * s, ph);
#pragma unroll
    for (int q = 0; q < NV; ++q) nn[q] = lds_f64(my0 + s * SB + q * TM_BOXB);
    const int r = rb + rel;
    rb = table ? sh.ptab[min(z + 1, np - 1)] : rb + S;
    if (!CHECK || r < plim) {
      const uint32_t cur = my0 + sc * SB;  // this plane's centre
      const uint32_t pid = lds_u8(id0 + sc * SB);
      SSCG_CHECK((int)pid < c.pat_np);
      const uint32_t va = pv0 + pid * (SS_MAX_NE * 8);
      const double2 v01 = lds_f64x2(va), v23 = lds_f64x2(va + 16), v45 = lds_f64x2(va + 32);
      const double v6 = lds_f64(va + 48);
      const double v[7] = {v01.x, v01.y, v23.x, v23.y, v45.x, v45.y, v6};
      double acc[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const uint32_t bx = cur + q * TM_BOXB;
        const double xb[7] = {p[q], lds_f64(bx - 8 * TM_W), lds_f64(bx - 8), cc[q],
                              lds_f64(bx + 8), lds_f64(bx + 8 * TM_W), nn[q]};
        double a = 0.0;
#pragma unroll
        for (int kk = 0; kk < 7; ++kk) {
          // EX: the off-centre values are 0 or +-1 (Ctx::tm_exact), their
          // products exact -- fma(v, x, a) is csr_matvec's a + v * x bit for bit
          if (EX && kk != 3)
            a = fma(v[kk], xb[kk], a);
          else
            a = __dadd_rn(a, __dmul_rn(v[kk], xb[kk]));
        }
        acc[q] = a;
      }
      if (L0 && r < n_own) {
        const double bi = lds_f64(b0 + sc * SB);
        const double t = __dsub_rn(bi, acc[0]);
        tt = fma(t, t, tt);
        rr = fma(cc[NV - 1], cc[NV - 1], rr);
      }
#pragma unroll
      for (int q = 0; q < NO; ++q) {
        if (q == NO - 1 && NO > 1 && r >= rlim) break;
        const double y2 = MU ? lds_f64(ym0 + sc * SB + q * 2048) : 0.0;
        const double w = tm_recur<UNIT>(acc[Q0 + q], cc[Q0 + q], y2, th, ga, mu, MU);
        SSCG_CHECK(r >= 0 && r < c.ld);
        zp.yo[q][r] = w;
        // exponent all ones (inf / NaN) carries into bit 31: checked once at the end
        badm |= (((unsigned)__double2hiint(w)) & 0x7ff00000u) + 0x00100000u;
      }
    }
    mbar_arrive_u32(empty0 + 8u * sc);
    sc = s;
    advance();
  };
  for (;;) {
    // the item's first stage: plane z0 - 1 (and the item id)
    tm_wait(full0 + 8u * s, ph);
    const int it = sh.sitem[s];
    if (it < 0) break;
    int cb, z0, z1;
    tm_item<L0>(c, it, ncb, cb, z0, z1);
    const int x0 = (cb % ntx) * 32, y0 = (cb / ntx) * 8;
    const int line = y0 + warp;
    const int rel = line * o + x0 + lane;  // row within its plane
    rb = table ? sh.ptab[z0] : z0 * S;
    // rows of this item: all below plim unless the tile passes the last line
    // or a plane lies at a ghost depth this level does not compute
    const bool all_in = line < lines && (table ? sh.sbase[s] : (z1 - 1) * S) + rel < plim;
    const bool live = line < lines;
    double pv[NV], cu[NV], nx[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) pv[q] = lds_f64(my0 + s * SB + q * TM_BOXB);
    mbar_arrive_u32(empty0 + 8u * s);
    advance();
    tm_wait(full0 + 8u * s, ph);
#pragma unroll
    for (int q = 0; q < NV; ++q) cu[q] = lds_f64(my0 + s * SB + q * TM_BOXB);
    int sc = s;
    advance();
    // planes in threes: the x[r - S], x[r], x[r + S] registers rotate by name
    if (all_in) {
      for (int z = z0; z < z1; z += 3) {
        step(std::false_type{}, pv, cu, nx, z, rel, sc);
        if (z + 1 >= z1) break;
        step(std::false_type{}, cu, nx, pv, z + 1, rel, sc);
        if (z + 2 >= z1) break;
        step(std::false_type{}, nx, pv, cu, z + 2, rel, sc);
      }
    } else {
      const int relc = live ? rel : INT32_MAX / 2;  // a dead line never computes
      for (int z = z0; z < z1; z += 3) {
        step(std::true_type{}, pv, cu, nx, z, relc, sc);
        if (z + 1 >= z1) break;
        step(std::true_type{}, cu, nx, pv, z + 1, relc, sc);
        if (z + 2 >= z1) break;
        step(std::true_type{}, nx, pv, cu, z + 2, relc, sc);
      }
    }
    mbar_arrive_u32(empty0 + 8u * sc);  // plane z1
  }
  const int bad = (badm & 0x80000000u) != 0;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&c.st->breakdown, 1);
  if (L0) {  // fixed-order partials of this CTA (static item assignment)
    tt = warp_sum(tt);
    rr = warp_sum(rr);
    if (lane == 0) {
      sh.red[0][warp] = tt;
      sh.red[1][warp] = rr;
    }
    consumers_bar();
    if (tid == 0) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        a += sh.red[0][w];
        b += sh.red[1][w];
      }
      c.part_t[blockIdx.x] = a;
      c.part_r[blockIdx.x] = b;
    }
  }
}

template <bool L0>
__global__ void __launch_bounds__(TM_THREADS, TM_MINB)
    k_level_tm(Ctx c, int l, ZmPtrs zp, const __grid_constant__ TmMaps maps) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (!L0 && l >= sbar) return;
  extern __shared__ __align__(128) unsigned char tsm[];
  constexpr int RING = Ring<L0>::R;
  __shared__ __align__(8) uint64_t full[RING], empty[RING];
  __shared__ int sitem[RING], sbase[RING];
  __shared__ double red[2][8];
  const int tid = threadIdx.x;
  const bool table = c.zm_base != nullptr;
  double* pval = reinterpret_cast<double*>(tsm);
  int* ptab = reinterpret_cast<int*>(tsm + (size_t)c.pat_np * SS_MAX_NE * 8);
  for (int j = tid; j < c.pat_np * SS_MAX_NE; j += blockDim.x) pval[j] = __ldg(c.ss_val + j);
  if (table)  // row base and plane index (the producer's TMA coordinate: no division per stage)
    for (int j = tid; j < c.zm_np; j += blockDim.x) {
      const int base = __ldg(c.zm_base + j);
      ptab[j] = base;
      ptab[c.zm_np + j] = base / (int)c.zm_S;
    }
  if (tid == 0) {
    for (int s = 0; s < RING; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  TmShared sh{full, empty, sitem, sbase, red, pval, ptab,
              tsm + tm_head_bytes(c.pat_np, c.zm_np, table)};
  TL_K(c, 0);
  TL_BEGIN(c, l);
  if (L0) {
    const bool do_r = sbar >= 2;
    if (st->prm.ga[0] == 1.0) {
      if (c.tm_exact)
        tm_body<3, true, 0, true>(c, 0, zp, maps, sh, false, do_r);
      else
        tm_body<3, true, 0, false>(c, 0, zp, maps, sh, false, do_r);
    } else {
      if (c.tm_exact)
        tm_body<3, true, 1, true>(c, 0, zp, maps, sh, false, do_r);
      else
        tm_body<3, true, 1, false>(c, 0, zp, maps, sh, false, do_r);
    }
    TL_END(c, 0);
    return;
  }
  const double ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const int rk = (ga == 1.0 ? 0 : 1) | (use_mu ? 2 : 0);
  const bool do_r = l < sbar - 1;
  const bool dyn = c.zm_ctr != nullptr && st->leja_on;
#define TM_RK(NV, EX)                                                      \
  switch (rk) {                                                            \
    case 0: tm_body<NV, false, 0, EX>(c, l, zp, maps, sh, dyn, do_r); break; \
    case 1: tm_body<NV, false, 1, EX>(c, l, zp, maps, sh, dyn, do_r); break; \
    case 2: tm_body<NV, false, 2, EX>(c, l, zp, maps, sh, dyn, do_r); break; \
    default: tm_body<NV, false, 3, EX>(c, l, zp, maps, sh, dyn, do_r); break; \
  }
  if (c.tm_exact) {
    if (do_r) {
      TM_RK(2, true)
    } else {
      TM_RK(1, true)
    }
  } else {
    if (do_r) {
      TM_RK(2, false)
    } else {
      TM_RK(1, false)
    }
  }
#undef TM_RK
  TL_END(c, l);
}

template <bool L0>
size_t tm_smem(const Ctx& c) {
  return tm_head_bytes(c.pat_np, c.zm_np, c.zm_base != nullptr) +
         (size_t)Ring<L0>::R * tm_stage_bytes(L0 ? 3 : 2, L0);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int encode(CUtensorMap* m, CUtensorMapDataType t, int rank, const void* base, const uint64_t* dims,
           const uint64_t* strides, const uint32_t* box) {
  auto fn = encode_fn();
  if (!fn) return sscg_fail(SSCG_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  cuuint64_t d[5], st[4];
  cuuint32_t b[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    if (i < rank - 1) st[i] = strides[i];
  }
  const CUresult r = fn(m, t, (cuuint32_t)rank, const_cast<void*>(base), d, st, b, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return sscg_fail(SSCG_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SSCG_OK;
}

}  // namespace

#ifdef MBAR_DEBUG
extern "C" int sscg_debug_mbar(unsigned* out8) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, g_mbar_dbg, sizeof(unsigned) * 8);
  const unsigned zero[8] = {};
  cudaMemcpyToSymbol(g_mbar_dbg, zero, sizeof(zero));
  return (int)cudaGetLastError();
}
#endif

// tensor maps of one plan: Y (4-D [col][plane][line][x] over every allocated
// column), x and b (3-D, level 0) and the 1-byte row ids (3-D)
int tm_make_maps(TmMaps* m, const double* Y, int64_t ld, int ncols, const double* x, const double* b,
                 const void* pid, int64_t o, int64_t S, int64_t planes, int64_t id_planes) {
  const uint64_t lines = (uint64_t)(S / o);
  {
    const uint64_t dims[4] = {(uint64_t)o, lines, (uint64_t)planes, (uint64_t)ncols};
    const uint64_t str[3] = {8ull * o, 8ull * S, 8ull * ld};
    const uint32_t box[4] = {TM_W, TM_H, 1, 1};
    int rc = encode(&m->y, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, Y, dims, str, box);
    if (rc) return rc;
  }
  const uint64_t dims3[3] = {(uint64_t)o, lines, (uint64_t)planes};
  const uint64_t str3[2] = {8ull * o, 8ull * S};
  {
    const uint32_t box[3] = {TM_W, TM_H, 1};
    int rc = encode(&m->x, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims3, str3, box);
    if (rc) return rc;
  }
  {
    const uint32_t box[3] = {32, 8, 1};
    int rc = encode(&m->b, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, b, dims3, str3, box);
    if (rc) return rc;
  }
  {
    const uint64_t dims[4] = {(uint64_t)o, lines, (uint64_t)planes, (uint64_t)ncols};
    const uint64_t str[3] = {8ull * o, 8ull * S, 8ull * ld};
    const uint32_t box[4] = {32, 8, 1, 1};
    int rc = encode(&m->y8, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, Y, dims, str, box);
    if (rc) return rc;
  }
  {
    const uint64_t dims[3] = {(uint64_t)o, lines, (uint64_t)id_planes};
    const uint64_t str[2] = {(uint64_t)o, (uint64_t)S};
    const uint32_t box[3] = {32, 8, 1};
    int rc = encode(&m->id, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, pid, dims, str, box);
    if (rc) return rc;
  }
  return SSCG_OK;
}

// CTAs per SM of level 0 / levels >= 1 (with the dynamic shared memory the
// plan's pattern table and plane table need)
void tm_occupancy(int pat_np, int zm_np, bool table, int* occ0, int* occ1) {
  const int lim = 200 * 1024;
  cudaFuncSetAttribute(k_level_tm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(k_level_tm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  const size_t head = tm_head_bytes(pat_np, zm_np, table);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ0, k_level_tm<true>, TM_THREADS,
                                                head + (size_t)TM_R0 * tm_stage_bytes(3, true));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ1, k_level_tm<false>, TM_THREADS,
                                                head + (size_t)TM_R * tm_stage_bytes(2, false));
}

void launch_level_tm(const Ctx& c, int level, int sigma, cudaStream_t s) {
  const ZmPtrs zp = zm_ptrs(c, level, sigma);
  if (level == 0)
    k_level_tm<true><<<c.red_n, TM_THREADS, tm_smem<true>(c), s>>>(c, 0, zp, *c.tm);
  else
    k_level_tm<false><<<c.tm_grid, TM_THREADS, tm_smem<false>(c), s>>>(c, level, zp, *c.tm);
}
