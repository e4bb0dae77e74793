// mpk.cu -- K_mpk: fp64 CSR matrix-powers kernel fused with the basis recurrence.
//
// Reference: basis.py:210-225 `_recurrence_columns` over lacore.py:25-34 `spmv`
// (scipy csr_matvec).  One launch per level l builds BOTH P_{l+1} and R_{l+1}
// from a single pass over A (the reference runs the P and R recurrences one after
// the other, reading A 2s-1 times per block; here A is read s times):
//
//   w = (A y_l - theta_l y_l) [- mu_{l-1} y_{l-1}] ;  y_{l+1} = w / gamma_l
//
// Rounding is the reference's, bit for bit: each row sum starts at 0.0 and adds
// val*x in stored order with separately rounded multiply and add (what
// csr_matvec compiles to), and the recurrence is evaluated op by op with
// __dmul_rn/__dsub_rn/__ddiv_rn (numpy's element-wise order, no contraction).
// Level 0 also forms the true residual t = b - A x (adaptive.py:138) and the
// partial sums of ||t||^2 and ||r||^2 (adaptive.py:139,158) on the same pass.
//
// Roofline (HBM-bound): per level 12 nnz + 4 (n+1) bytes of A plus
// 16 n per generated column (+8 n with the Chebyshev two-back term).
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
template <int NV>
__device__ __forceinline__ void row_dot(const int* __restrict__ col, const double* __restrict__ val,
                                        int beg, int end, const double* const* __restrict__ xs,
                                        double* acc) {
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  int jj = beg;
  for (; jj + 4 <= end; jj += 4) {
    int c0 = __ldg(col + jj), c1 = __ldg(col + jj + 1), c2 = __ldg(col + jj + 2),
        c3 = __ldg(col + jj + 3);
    double v0 = __ldg(val + jj), v1 = __ldg(val + jj + 1), v2 = __ldg(val + jj + 2),
           v3 = __ldg(val + jj + 3);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double x0 = __ldg(xs[q] + c0), x1 = __ldg(xs[q] + c1), x2 = __ldg(xs[q] + c2),
             x3 = __ldg(xs[q] + c3);
      double a = acc[q];
      a = __dadd_rn(a, __dmul_rn(v0, x0));
      a = __dadd_rn(a, __dmul_rn(v1, x1));
      a = __dadd_rn(a, __dmul_rn(v2, x2));
      a = __dadd_rn(a, __dmul_rn(v3, x3));
      acc[q] = a;
    }
  }
  for (; jj < end; ++jj) {
    int c0 = __ldg(col + jj);
    double v0 = __ldg(val + jj);
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v0, __ldg(xs[q] + c0)));
  }
}

// one recurrence step, reference order: ((Ay - th*y) - mu*y2) / ga
__device__ __forceinline__ double recur(double ay, double y, double y2, double th, double ga,
                                        double mu, bool use_mu) {
  double w = __dsub_rn(ay, __dmul_rn(th, y));
  if (use_mu) w = __dsub_rn(w, __dmul_rn(mu, y2));
  return __ddiv_rn(w, ga);
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  uint32_t spins = 0;
  while (!done) {
    if (++spins > (1u << 26)) __trap();  // a lost transaction must fail, not hang
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

template <int NV>
__device__ __forceinline__ void row_dot_s(const TileStage& ts, int beg, int end,
                                          const double* const* __restrict__ xs, double* acc) {
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  const double* vv = ts.val - ts.beg_v;
  const int* cc = ts.col - ts.beg_c;
  int jj = beg;
  for (; jj + 2 <= end; jj += 2) {
    const int c0 = cc[jj], c1 = cc[jj + 1];
    const double v0 = vv[jj], v1 = vv[jj + 1];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const double x0 = __ldg(xs[q] + c0), x1 = __ldg(xs[q] + c1);
      acc[q] = __dadd_rn(__dadd_rn(acc[q], __dmul_rn(v0, x0)), __dmul_rn(v1, x1));
    }
  }
  if (jj < end) {
    const int c0 = cc[jj];
    const double v0 = vv[jj];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v0, __ldg(xs[q] + c0)));
  }
}

__global__ void __launch_bounds__(MT_ROWS) k_level0_staged(Ctx c) {
  __shared__ double sm[MT_ROWS / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  const double* P0 = c.Y;
  double* P1 = c.Y + c.ld;
  const double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
  double* R1 = c.Y + (int64_t)(sigma + 2) * c.ld;
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int64_t n_own = c.n_own, rlim = lvl_r_rows(c, sigma, 0);
  staged_rows(c, lvl_p_rows(c, sigma, 0), [&](int64_t i, const TileStage& ts) {
    const int beg = c.rp[i], end = c.rp[i + 1];
    const double p = P0[i], r = R0[i];
    double acc[3];
    const double* xs[3] = {c.x, P0, R0};
    if (do_r)
      row_dot_s<3>(ts, beg, end, xs, acc);
    else
      row_dot_s<2>(ts, beg, end, xs, acc);
    if (i < n_own) {
      const double t = __dsub_rn(c.b[i], acc[0]);
      tt = fma(t, t, tt);
      rr = fma(r, r, rr);
    }
    const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
    P1[i] = wp;
    bad |= !finite(wp);
    if (do_r && i < rlim) {
      const double wr = recur(acc[2], r, 0.0, th, ga, 0.0, false);
      R1[i] = wr;
      bad |= !finite(wr);
    }
  });
  tt = block_sum<MT_ROWS>(tt, sm);
  rr = block_sum<MT_ROWS>(rr, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = tt;
    c.part_r[blockIdx.x] = rr;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

__global__ void __launch_bounds__(MT_ROWS) k_level_staged(Ctx c, int l) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const double* Pl = c.Y + (int64_t)l * c.ld;
  const double* Pm = Pl - c.ld;
  double* Pn = c.Y + (int64_t)(l + 1) * c.ld;
  const double* Rl = c.Y + (int64_t)(sigma + 1 + l) * c.ld;
  const double* Rm = Rl - c.ld;
  double* Rn = c.Y + (int64_t)(sigma + 2 + l) * c.ld;
  int bad = 0;
  const int64_t rlim = lvl_r_rows(c, sigma, l);
  staged_rows(c, lvl_p_rows(c, sigma, l), [&](int64_t i, const TileStage& ts) {
    const int beg = c.rp[i], end = c.rp[i + 1];
    double acc[2];
    const double* xs[2] = {Pl, Rl};
    const bool rr = do_r && i < rlim;
    if (rr)
      row_dot_s<2>(ts, beg, end, xs, acc);
    else
      row_dot_s<1>(ts, beg, end, xs, acc);
    const double wp = recur(acc[0], Pl[i], use_mu ? Pm[i] : 0.0, th, ga, mu, use_mu);
    Pn[i] = wp;
    bad |= !finite(wp);
    if (rr) {
      const double wr = recur(acc[1], Rl[i], use_mu ? Rm[i] : 0.0, th, ga, mu, use_mu);
      Rn[i] = wr;
      bad |= !finite(wr);
    }
  });
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// ---------------------------------------------------------------------------
// Level 0 of an outer loop: t = b - A x (norm partial), ||r0||^2 partial,
// P_1 and (if s_bar >= 2) R_1.
__global__ void __launch_bounds__(ROWS_PER_CTA) k_level0(Ctx c) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  const double* P0 = c.Y;
  double* P1 = c.Y + c.ld;
  const double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
  double* R1 = c.Y + (int64_t)(sigma + 2) * c.ld;
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int64_t n_own = c.n_own, plim = lvl_p_rows(c, sigma, 0), rlim = lvl_r_rows(c, sigma, 0);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < plim; i += stride) {
    const int beg = c.rp[i], end = c.rp[i + 1];
    const double p = P0[i], r = R0[i];
    double acc[3];
    if (do_r) {
      const double* xs[3] = {c.x, P0, R0};
      row_dot<3>(c.col, c.val, beg, end, xs, acc);
    } else {
      const double* xs[2] = {c.x, P0};
      row_dot<2>(c.col, c.val, beg, end, xs, acc);
    }
    if (i < n_own) {
      const double t = __dsub_rn(c.b[i], acc[0]);
      tt = fma(t, t, tt);
      rr = fma(r, r, rr);
    }
    const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
    P1[i] = wp;
    bad |= !finite(wp);
    if (do_r && i < rlim) {
      const double wr = recur(acc[2], r, 0.0, th, ga, 0.0, false);
      R1[i] = wr;
      bad |= !finite(wr);
    }
  }
  tt = block_sum<ROWS_PER_CTA>(tt, sm);
  rr = block_sum<ROWS_PER_CTA>(rr, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = tt;
    c.part_r[blockIdx.x] = rr;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// Level l >= 1: P_{l+1} (l < s_bar) and R_{l+1} (l < s_bar - 1).
template <bool DO_R>
__device__ __forceinline__ int level_rows(const Ctx& c, int l, int sigma, double th, double ga,
                                          double mu, bool use_mu) {
  const int64_t plim = lvl_p_rows(c, sigma, l), rlim = lvl_r_rows(c, sigma, l);
  const double* Pl = c.Y + (int64_t)l * c.ld;
  const double* Pm = Pl - c.ld;
  double* Pn = c.Y + (int64_t)(l + 1) * c.ld;
  const double* Rl = c.Y + (int64_t)(sigma + 1 + l) * c.ld;
  const double* Rm = Rl - c.ld;
  double* Rn = c.Y + (int64_t)(sigma + 2 + l) * c.ld;
  int bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < plim; i += stride) {
    const int beg = c.rp[i], end = c.rp[i + 1];
    const bool rr = DO_R && i < rlim;
    double acc[2];
    if (rr) {
      const double* xs[2] = {Pl, Rl};
      row_dot<2>(c.col, c.val, beg, end, xs, acc);
    } else {
      const double* xs[1] = {Pl};
      row_dot<1>(c.col, c.val, beg, end, xs, acc);
    }
    const double wp = recur(acc[0], Pl[i], use_mu ? Pm[i] : 0.0, th, ga, mu, use_mu);
    Pn[i] = wp;
    bad |= !finite(wp);
    if (rr) {
      const double wr = recur(acc[1], Rl[i], use_mu ? Rm[i] : 0.0, th, ga, mu, use_mu);
      Rn[i] = wr;
      bad |= !finite(wr);
    }
  }
  return bad;
}

__global__ void __launch_bounds__(ROWS_PER_CTA) k_level(Ctx c, int l) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  int bad = (l < sbar - 1) ? level_rows<true>(c, l, sigma, th, ga, mu, use_mu)
                           : level_rows<false>(c, l, sigma, th, ga, mu, use_mu);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// Initial residual (adaptive.py:121-123): r = b - A x0 into Y[:, sigma+1], p = r into
// Y[:, 0], x = x0; partial ||b||^2 into part_t (for nb, adaptive.py:118).
__global__ void __launch_bounds__(ROWS_PER_CTA) k_init_residual(Ctx c, const double* x0) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const int sigma = c.cfg->sigma;
  double* P0 = c.Y;
  double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
  double bb = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.lvl_rows[SMAX]; i += stride) {
    if (i >= c.n_own) {  // ghost rows: x from x0; p, r arrive with the first halo exchange
      c.x[i] = x0[i];
      continue;
    }
    double acc[1];
    const double* xs[1] = {x0};
    row_dot<1>(c.col, c.val, c.rp[i], c.rp[i + 1], xs, acc);
    const double bi = c.b[i];
    const double r = __dsub_rn(bi, acc[0]);
    R0[i] = r;
    P0[i] = r;
    c.x[i] = x0[i];
    bb = fma(bi, bi, bb);
  }
  bb = block_sum<ROWS_PER_CTA>(bb, sm);
  if (threadIdx.x == 0) c.part_t[blockIdx.x] = bb;
}

// Full-trace diagnostics (adaptive.py:205-215): tv = b - A x_j; partials of
// ||tv||^2, ||r_j||^2, ||tv - r_j||^2.  x_j / r_j were formed by k_diag_form.
__global__ void __launch_bounds__(ROWS_PER_CTA) k_diag_resid(Ctx c, int j) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  if (j >= c.st->diag_n) return;
  double s_t = 0.0, s_r = 0.0, s_g = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n_own; i += stride) {
    double acc[1];
    const double* xs[1] = {c.xj};
    row_dot<1>(c.col, c.val, c.rp[i], c.rp[i + 1], xs, acc);
    const double tv = __dsub_rn(c.b[i], acc[0]);
    const double r = c.rj[i];
    const double g = __dsub_rn(tv, r);
    s_t = fma(tv, tv, s_t);
    s_r = fma(r, r, s_r);
    s_g = fma(g, g, s_g);
  }
  s_t = block_sum<ROWS_PER_CTA>(s_t, sm);
  s_r = block_sum<ROWS_PER_CTA>(s_r, sm);
  s_g = block_sum<ROWS_PER_CTA>(s_g, sm);
  if (threadIdx.x == 0) {
    c.part_d[blockIdx.x] = s_t;
    c.part_d[RED_BLOCKS + blockIdx.x] = s_r;
    c.part_d[2 * RED_BLOCKS + blockIdx.x] = s_g;
  }
}

// ---- unit-entry kernels (explicit parameters, no solver state) ------------
__global__ void __launch_bounds__(ROWS_PER_CTA)
    k_spmv(const int* __restrict__ rp, const int* __restrict__ col,
           const double* __restrict__ val, int64_t n, const double* __restrict__ x, double* y) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double acc[1];
    const double* xs[1] = {x};
    row_dot<1>(col, val, rp[i], rp[i + 1], xs, acc);
    y[i] = acc[0];
  }
}

// one level of a standalone block build (columns: P at 0..s, R at s+1..2s)
__global__ void __launch_bounds__(ROWS_PER_CTA)
    k_block_level(const int* __restrict__ rp, const int* __restrict__ col,
                  const double* __restrict__ val, int64_t n, int64_t ld, double* Y, int s, int l,
                  double th, double ga, double mu, int* breakdown) {
  const bool use_mu = (l >= 1) && !(mu == 0.0);
  const bool do_p = l < s, do_r = l < s - 1;
  const double* Pl = Y + (int64_t)l * ld;
  double* Pn = Y + (int64_t)(l + 1) * ld;
  const double* Rl = Y + (int64_t)(s + 1 + l) * ld;
  double* Rn = Y + (int64_t)(s + 2 + l) * ld;
  int bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int beg = rp[i], end = rp[i + 1];
    double acc[2];
    const double* xs[2] = {Pl, Rl};
    row_dot<2>(col, val, beg, end, xs, acc);
    if (do_p) {
      double w = recur(acc[0], Pl[i], use_mu ? Pl[i - ld] : 0.0, th, ga, mu, use_mu);
      Pn[i] = w;
      bad |= !finite(w);
    }
    if (do_r) {
      double w = recur(acc[1], Rl[i], use_mu ? Rl[i - ld] : 0.0, th, ga, mu, use_mu);
      Rn[i] = w;
      bad |= !finite(w);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(breakdown, 1);
}

inline int grid_rows(int64_t n) {
  int64_t g = (n + ROWS_PER_CTA - 1) / ROWS_PER_CTA;
  if (g > RED_BLOCKS) g = RED_BLOCKS;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

// The row-streaming kernels always launch RED_BLOCKS CTAs (grid-stride) so the
// partial-sum arrays have a fixed length and the reductions a fixed order.
size_t staged_smem_bytes(int cap) { return MT_STAGES * stage_bytes(cap); }

// The attribute is per kernel and process-wide, and several plans (ranks of a
// virtual group, different matrices) may coexist: raise it once to the staging
// ceiling instead of to one plan's tile size.
void staged_prepare(int cap) {
  (void)cap;
  const int bytes = 200 * 1024;
  cudaFuncSetAttribute(k_level0_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_level_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

int staged_ctas_per_sm(int cap) {
  int a = 0, b = 0;
  const size_t bytes = staged_smem_bytes(cap);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_level0_staged, MT_ROWS, bytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_level_staged, MT_ROWS, bytes);
  return a < b ? a : b;
}

void launch_init_residual(const Ctx& c, const double* x0, cudaStream_t s) {
  k_init_residual<<<c.red_n, ROWS_PER_CTA, 0, s>>>(c, x0);
}
void launch_level(const Ctx& c, int level, cudaStream_t s) {
  if (c.stage_cap > 0) {
    const size_t bytes = staged_smem_bytes(c.stage_cap);
    if (level == 0)
      k_level0_staged<<<c.red_n, MT_ROWS, bytes, s>>>(c);
    else
      k_level_staged<<<c.red_n, MT_ROWS, bytes, s>>>(c, level);
    return;
  }
  if (level == 0)
    k_level0<<<c.red_n, ROWS_PER_CTA, 0, s>>>(c);
  else
    k_level<<<c.red_n, ROWS_PER_CTA, 0, s>>>(c, level);
}
void launch_spmv(const int* rp, const int* col, const double* val, int64_t n, const double* x,
                 double* y, cudaStream_t s) {
  k_spmv<<<grid_rows(n), ROWS_PER_CTA, 0, s>>>(rp, col, val, n, x, y);
}
void launch_block_levels(const int* rp, const int* col, const double* val, int64_t n, int64_t ld,
                         double* Y, int s, const double* th, const double* ga, const double* mu,
                         int* breakdown, cudaStream_t st) {
  for (int l = 0; l < s; ++l)
    k_block_level<<<grid_rows(n), ROWS_PER_CTA, 0, st>>>(rp, col, val, n, ld, Y, s, l, th[l], ga[l],
                                                          l >= 1 ? mu[l - 1] : 0.0, breakdown);
}
void launch_diag_resid(const Ctx& c, int j, cudaStream_t s) {
  k_diag_resid<<<c.red_n, ROWS_PER_CTA, 0, s>>>(c, j);
}
