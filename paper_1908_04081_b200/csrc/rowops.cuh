// rowops.cuh -- device building blocks of the row-streaming kernels (matrix
// powers, HSCG): deterministic reductions, csr_matvec-exact row sums from CSR,
// TMA-staged CSR tiles or the pattern-compressed operator, the basis
// recurrence step.  Header-only, internal linkage (one copy per .cu).
#pragma once
#include <cstdio>

#include "internal.cuh"

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block sum (fixed shuffle tree + fixed smem order); result in thread 0
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sm) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sm[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) r += sm[i];
  }
  __syncthreads();
  return r;
}

// csr_matvec row sum for NV right-hand sides sharing one pass over the row
#ifndef CSR_CHUNK
#define CSR_CHUNK 4
#endif
// csr_matvec row sum from global CSR (direct kernels).  Chunks of CSR_CHUNK
// entries: the next chunk's col/val loads are issued before this chunk's
// gathers are consumed, so a long row costs about one load round per chunk
// instead of two; adds in stored order (a lane past the end adds nothing).
template <int NV>
__device__ __forceinline__ void row_dot(const int* __restrict__ col, const double* __restrict__ val,
                                        int beg, int end, const double* const* __restrict__ xs,
                                        double* acc) {
  constexpr int K = CSR_CHUNK;
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  if (beg >= end) return;
  int c[K];
  double v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int j = beg + k < end ? beg + k : end - 1;
    c[k] = __ldg(col + j);
    v[k] = __ldg(val + j);
  }
  for (int jj = beg; jj < end; jj += K) {
    double x[NV][K];
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int k = 0; k < K; ++k) x[q][k] = __ldg(xs[q] + c[k]);
    const int m = end - jj;
    double vc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) vc[k] = v[k];
    if (jj + K < end) {  // prefetch the next chunk
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int j = jj + K + k < end ? jj + K + k : end - 1;
        c[k] = __ldg(col + j);
        v[k] = __ldg(val + j);
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (k < m)
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(vc[k], x[q][k]));
  }
}

// one recurrence step, reference order: ((Ay - th*y) - mu*y2) / ga.  The IEEE
// quotient w / 1.0 is w exactly (NaN, +-0 and +-inf included), so the unit
// scaling of the Newton and monomial bases skips the division sequence.
__device__ __forceinline__ double recur(double ay, double y, double y2, double th, double ga,
                                        double mu, bool use_mu) {
  double w = __dsub_rn(ay, __dmul_rn(th, y));
  if (use_mu) w = __dsub_rn(w, __dmul_rn(mu, y2));
  return ga == 1.0 ? w : __ddiv_rn(w, ga);
}

__device__ __forceinline__ bool finite(double v) { return isfinite(v); }

// ---------------------------------------------------------------------------
// TMA-staged CSR tiles.  Persistent CTAs walk MT_ROWS-row tiles; the tile's
// contiguous col/val segment is moved global->shared by cp.async.bulk (one
// elected thread, mbarrier completion), double-buffered, so the CSR stream is
// in flight while the previous tile's rows are computed.  Row sums still run
// sequentially in stored order from shared memory: bit-identical to csr_matvec.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// bulk L2 prefetch (TMA unit, no registers, no completion tracking)
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
// Row-streaming pattern kernels: the CTA's rows of the NEXT grid-stride
// iteration first touch the input vectors around row + pf_off (the largest
// positive column offset: a stencil's plane ahead).  One thread per CTA asks
// the TMA unit to pull those 256-row windows into L2 now, so the gathers of
// the next iteration hit L2 instead of waiting on HBM (more bytes in flight
// per SM than the threads' own loads can keep).
template <int NV>
__device__ __forceinline__ void prefetch_next(const Ctx& c, int64_t i, int64_t stride,
                                              const double* const* xs) {
  if (c.pf_off == 0 || threadIdx.x != 0) return;
  int64_t r0 = i + (int64_t)c.pf_ahead * stride + c.pf_off;
  r0 &= ~(int64_t)1;
  if (r0 < 0 || r0 + ROWS_PER_CTA > c.ld) return;
#pragma unroll
  for (int q = 0; q < NV; ++q) l2_prefetch(xs[q] + r0, ROWS_PER_CTA * 8);
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
#ifdef MBAR_DEBUG
// debug side builds: a timed-out wait records (count, block, thread, barrier,
// parity) here and gives up instead of trapping, so the host can read it
__device__ unsigned g_mbar_dbg[8];
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  uint32_t spins = 0;
  while (!done) {
#ifdef MBAR_DEBUG
    if (++spins > (1u << 20)) {
      if (atomicAdd(&g_mbar_dbg[0], 1u) == 0) {
        g_mbar_dbg[1] = blockIdx.x;
        g_mbar_dbg[2] = threadIdx.x;
        g_mbar_dbg[3] = smem_u32(bar);
        g_mbar_dbg[4] = parity;
      }
      return;
    }
#else
    if (++spins > (1u << 26)) __trap();  // a lost transaction must fail, not hang
#endif
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

struct TileStage {
  const double* val;  // shared: val[beg_v ..)
  const int* col;     // shared: col[beg_c ..)
  int beg_v, beg_c;
};

// stage layout: [cap + 2 doubles of val][cap + 4 ints of col], 16-byte aligned
__host__ __device__ __forceinline__ size_t stage_bytes(int cap) {
  return ((size_t)(cap + 2) * 8 + (size_t)(cap + 4) * 4 + 15) / 16 * 16;
}

// Runs fn(row, TileStage&) over rows [0, nrows) tile by tile.
template <class Fn>
__device__ __forceinline__ void staged_rows(const Ctx& c, int64_t nrows, Fn&& fn) {
  extern __shared__ __align__(16) unsigned char msm[];
  __shared__ __align__(8) uint64_t bars[MT_STAGES];
  __shared__ int tb[MT_STAGES][2];
  const int cap = c.stage_cap;
  const size_t sb = stage_bytes(cap);
  const int64_t ntiles = (nrows + MT_ROWS - 1) / MT_ROWS;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < MT_STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t tile, int s) {  // thread 0 only
    const int64_t r0 = tile * MT_ROWS;
    const int64_t r1 = r0 + MT_ROWS < nrows ? r0 + MT_ROWS : nrows;
    const int beg = c.rp[r0], end = c.rp[r1];
    const int bv = beg & ~1, bc = beg & ~3;
    const uint32_t nbv = (uint32_t)(((end - bv) * 8 + 15) / 16 * 16);
    const uint32_t nbc = (uint32_t)(((end - bc) * 4 + 15) / 16 * 16);
    tb[s][0] = bv;
    tb[s][1] = bc;
    unsigned char* base = msm + (size_t)s * sb;
    mbar_arrive_tx(&bars[s], nbv + nbc);
    if (nbv) bulk_g2s(base, c.val + bv, nbv, &bars[s]);
    if (nbc) bulk_g2s(base + (size_t)(cap + 2) * 8, c.col + bc, nbc, &bars[s]);
  };
  int64_t k = 0;
  if (tid == 0)
    for (int s = 0; s < MT_STAGES; ++s) {
      const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
      if (t < ntiles) issue(t, s);
    }
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
    const int s = (int)(k % MT_STAGES);
    mbar_wait(&bars[s], (uint32_t)((k / MT_STAGES) & 1));
    TileStage ts;
    unsigned char* base = msm + (size_t)s * sb;
    ts.val = reinterpret_cast<const double*>(base);
    ts.col = reinterpret_cast<const int*>(base + (size_t)(cap + 2) * 8);
    ts.beg_v = tb[s][0];
    ts.beg_c = tb[s][1];
    const int64_t i = tile * MT_ROWS + tid;
    if (i < nrows) fn(i, ts);
    __syncthreads();  // stage s free again
    if (tid == 0) {
      const int64_t t = tile + (int64_t)MT_STAGES * gridDim.x;
      if (t < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(t, s);
      }
    }
  }
}

// gathers of vectors that are read-only for the whole launch
struct LdNc {
  static __device__ __forceinline__ double ld(const double* p) { return __ldg(p); }
};
#ifndef ROW_BATCH
#define ROW_BATCH 4
#endif
// Row sums from a staged tile.  The gathers of a chunk of up to B nonzeros are
// all issued before the chunk is accumulated -- B x NV loads in flight per
// thread instead of a chain of dependent load rounds -- and the adds then run
// strictly in stored order (a lane past the row end adds nothing, not +0.0,
// so even the sign of a zero sum is csr_matvec's).
template <int NV, class LD = LdNc, int B = (NV >= 3 ? (ROW_BATCH + 1) / 2 : ROW_BATCH)>
__device__ __forceinline__ void row_dot_s(const TileStage& ts, int beg, int end,
                                          const double* const* __restrict__ xs, double* acc) {
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  const double* vv = ts.val - ts.beg_v;
  const int* cc = ts.col - ts.beg_c;
  for (int jj = beg; jj < end; jj += B) {
    const int m = end - jj;
    int cb[B];
#pragma unroll
    for (int k = 0; k < B; ++k) cb[k] = cc[jj + (k < m ? k : 0)];
    double xb[NV][B];
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int k = 0; k < B; ++k) xb[q][k] = LD::ld(xs[q] + cb[k]);
#pragma unroll
    for (int k = 0; k < B; ++k) {
      if (k < m) {
        const double v = vv[jj + k];
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v, xb[q][k]));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Pattern-compressed level kernels.  A stencil-like operator has few distinct
// rows up to translation: the pattern table (offsets relative to the row,
// values, in stored order) sits in shared memory and each row streams only
// its 1- or 2-byte pattern id, so a level moves ~33 bytes per row (ids, the
// two input and two output basis entries) instead of ~120 with CSR.  The row
// sum is the same sequence of rounded multiply-adds as csr_matvec -- same
// columns, values and order -- hence bit-identical to the CSR kernels.
__host__ __device__ __forceinline__ size_t pattern_smem_bytes_dev(int np, int ne) {
  return (size_t)ne * 12 + (size_t)(np + 1) * 4;
}

struct PatSmem {
  const double* val;
  const int* off;
  const int* ptr;
};

// table layout in dynamic shared memory: [val ne][ptr np+1][off ne]
__device__ __forceinline__ PatSmem load_patterns(const Ctx& c) {
  extern __shared__ __align__(16) double psm[];
  double* sv = psm;
  int* sp = reinterpret_cast<int*>(sv + c.pat_ne);
  int* so = sp + c.pat_np + 1;
  for (int j = threadIdx.x; j < c.pat_ne; j += blockDim.x) {
    sv[j] = __ldg(c.pat_val + j);
    so[j] = __ldg(c.pat_off + j);
  }
  for (int j = threadIdx.x; j <= c.pat_np; j += blockDim.x) sp[j] = __ldg(c.pat_ptr + j);
  __syncthreads();
  return PatSmem{sv, so, sp};
}

template <typename ID>
__device__ __forceinline__ int row_pattern(const Ctx& c, int64_t i) {
  return (int)__ldg(reinterpret_cast<const ID*>(c.pid) + i);
}

#ifndef PAT_BATCH
#define PAT_BATCH 8
#endif
template <int NV, int B = (NV >= 3 ? PAT_BATCH / 2 : PAT_BATCH)>
__device__ __forceinline__ void row_dot_p(const PatSmem& T, int b, int e, int i,
                                          const double* const* __restrict__ xs, double* acc) {
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  for (int jj = b; jj < e; jj += B) {
    const int m = e - jj;
    int cb[B];
#pragma unroll
    for (int k = 0; k < B; ++k) cb[k] = i + T.off[jj + (k < m ? k : 0)];
    double xb[NV][B];
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
      for (int k = 0; k < B; ++k) xb[q][k] = __ldg(xs[q] + cb[k]);
#pragma unroll
    for (int k = 0; k < B; ++k) {
      if (k < m) {
        const double v = T.val[jj + k];
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v, xb[q][k]));
      }
    }
  }
}

// Superset-mask form (Ctx::ss_*): the table as per-pattern masks over the
// sorted union of offsets plus per-slot values.  The union offsets are kernel
// parameters, so the row loop is fully unrolled: per present slot one address,
// NV gathers, then the adds in slot order = the stored order of the row (a
// pattern's offsets are a subsequence of the sorted union), i.e. the same
// rounded multiply-adds as csr_matvec.  Table in shared memory:
// [val np x SS_MAX_NE][mask np].
// [val np x SS_MAX_NE][mask np][pad to 16][eoff np x int4]
__host__ __device__ __forceinline__ size_t ss_eoff_offset(int np) {
  return ((size_t)np * SS_MAX_NE * 8 + (size_t)np * 4 + 15) / 16 * 16;
}
__host__ __device__ __forceinline__ size_t ss_smem_bytes_dev(int np) {
  return ss_eoff_offset(np) + (size_t)np * 16;
}

struct SsSmem {
  const double* val;
  const unsigned* mask;
  const int4* eoff;  // per pattern: the offsets of the union's middle slots (plane
                     // march: slots 1, 2, NE-3, NE-2 of 7; 1, 3 of 5), 0 where absent
};

__device__ __forceinline__ SsSmem load_ss(const Ctx& c) {
  extern __shared__ __align__(16) double psm[];
  double* sv = psm;
  unsigned* sm = reinterpret_cast<unsigned*>(sv + (size_t)c.pat_np * SS_MAX_NE);
  int4* se = reinterpret_cast<int4*>(reinterpret_cast<char*>(psm) + ss_eoff_offset(c.pat_np));
  for (int j = threadIdx.x; j < c.pat_np * SS_MAX_NE; j += blockDim.x) sv[j] = __ldg(c.ss_val + j);
  const int ne = c.ss_ne;
  for (int j = threadIdx.x; j < c.pat_np; j += blockDim.x) {
    const unsigned m = __ldg(c.ss_mask + j);
    sm[j] = m;
    // middle slots of a symmetric 7- or 5-slot union (the -S / 0 / +S slots
    // of the march come from registers); an absent slot reads offset 0
    int4 e = make_int4(0, 0, 0, 0);
    if (ne == 7) {
      e.x = (m >> 1) & 1u ? c.ss_off[1] : 0;
      e.y = (m >> 2) & 1u ? c.ss_off[2] : 0;
      e.z = (m >> 4) & 1u ? c.ss_off[4] : 0;
      e.w = (m >> 5) & 1u ? c.ss_off[5] : 0;
    } else if (ne == 5) {
      e.x = (m >> 1) & 1u ? c.ss_off[1] : 0;
      e.y = (m >> 3) & 1u ? c.ss_off[3] : 0;
    }
    se[j] = e;
  }
  __syncthreads();
  return SsSmem{sv, sm, se};
}

// The adds run over every slot: an absent slot contributes 0.0 * 0.0 = +0.0,
// and adding +0.0 is exact for every partial sum csr_matvec can hold (a sum
// that starts at +0.0 is never -0.0 under round-to-nearest), so the result is
// bit-identical to skipping the slot.  Only the gathers are predicated (an
// absent slot's column may lie outside the vector).
template <int NV, int NE>
__device__ __forceinline__ void row_dot_m(const Ctx& c, const SsSmem& S, int pid, int64_t i,
                                          const double* const* __restrict__ xs, double* acc) {
  const unsigned m = S.mask[pid];
  const double2* v2 = reinterpret_cast<const double2*>(S.val + pid * SS_MAX_NE);
  const double* xi[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) xi[q] = xs[q] + i;  // row base; slot k reads xi[q][off_k]
  double xb[NV][NE];
#pragma unroll
  for (int k = 0; k < NE; ++k) {
#pragma unroll
    for (int q = 0; q < NV; ++q) xb[q][k] = 0.0;
    if (m & (1u << k)) {
      const int o = c.ss_off[k];
#pragma unroll
      for (int q = 0; q < NV; ++q) xb[q][k] = __ldg(xi[q] + o);
    }
  }
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
#pragma unroll
  for (int k2 = 0; k2 < (NE + 1) / 2; ++k2) {
    const double2 vv = v2[k2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = 2 * k2 + h;
      if (k < NE) {
        const double v = h ? vv.y : vv.x;
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v, xb[q][k]));
      }
    }
  }
}

}  // namespace
