// mpk.cu -- K_mpk: fp64 matrix-powers kernels fused with the basis recurrence.
//
// Kernel families (plan.cu picks one per operator; all bit-identical):
//   k_level0_zm / k_level_zm      plane march over a pattern-compressed stencil
//                                 (the default for c1 c3 c5: 1-byte row ids)
//   k_level0_ss / k_level_ss      superset-mask pattern rows (small strides)
//   k_level0_pat / k_level_pat    table-walk pattern rows (any pattern operator)
//   k_level0_vs / k_level_vs      value stream: stencil structure, row-varying
//                                 values (c4), no column indices
//   k_level0_staged / k_level_staged, k_level0 / k_level   general CSR
// (variants measured slower in round 1 -- wavefront passes, TMA windows, row
// pairs, a barrier-per-plane tile march, a split level 0 -- are described in
// DESIGN.md 4a / 4b and live in git history, not here)
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
// Roofline (HBM-bound): per level 12 nnz + 4 (n+1) bytes of A for
// CSR (1-2 n for a pattern operator, 8 ne n for a value stream) plus 16 n per
// generated column (+8 n with the Chebyshev two-back term).
#include "internal.cuh"
#include "rowops.cuh"

namespace {

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

template <typename ID>
__global__ void __launch_bounds__(ROWS_PER_CTA) k_level0_pat(Ctx c) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const PatSmem T = load_patterns(c);
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
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int pid_next = i < plim ? row_pattern<ID>(c, i) : 0;  // ids one row ahead
  for (; i < plim; i += stride) {
    const int pid = pid_next;
    {
      const double* pf[3] = {c.x, P0, R0};
      prefetch_next<3>(c, i, stride, pf);
    }
    if (i + stride < plim) pid_next = row_pattern<ID>(c, i + stride);
    const int b = T.ptr[pid], e = T.ptr[pid + 1];
    const double p = P0[i], r = R0[i];
    double acc[3];
    const double* xs[3] = {c.x, P0, R0};
    if (do_r)
      row_dot_p<3>(T, b, e, (int)i, xs, acc);
    else
      row_dot_p<2>(T, b, e, (int)i, xs, acc);
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

// (an explicit min-blocks of 1 lets ptxas take ~85 registers: 2 CTAs/SM;
// 0 = no min-blocks hint)
#ifndef PAT_MINB
#define PAT_MINB 0
#endif
#if PAT_MINB > 0
#define PAT_LB __launch_bounds__(ROWS_PER_CTA, PAT_MINB)
#else
#define PAT_LB __launch_bounds__(ROWS_PER_CTA)
#endif
template <typename ID>
__global__ void PAT_LB k_level_pat(Ctx c, int l) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const PatSmem T = load_patterns(c);
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
  const int64_t plim = lvl_p_rows(c, sigma, l), rlim = lvl_r_rows(c, sigma, l);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int pid_next = i < plim ? row_pattern<ID>(c, i) : 0;  // ids one row ahead
  for (; i < plim; i += stride) {
    const int pid = pid_next;
    {
      const double* pf[2] = {Pl, Rl};
      prefetch_next<2>(c, i, stride, pf);
    }
    if (i + stride < plim) pid_next = row_pattern<ID>(c, i + stride);
    const int b = T.ptr[pid], e = T.ptr[pid + 1];
    double acc[2];
    const double* xs[2] = {Pl, Rl};
    const bool rrow = do_r && i < rlim;
    if (rrow)
      row_dot_p<2>(T, b, e, (int)i, xs, acc);
    else
      row_dot_p<1>(T, b, e, (int)i, xs, acc);
    const double wp = recur(acc[0], Pl[i], use_mu ? Pm[i] : 0.0, th, ga, mu, use_mu);
    Pn[i] = wp;
    bad |= !finite(wp);
    if (rrow) {
      const double wr = recur(acc[1], Rl[i], use_mu ? Rm[i] : 0.0, th, ga, mu, use_mu);
      Rn[i] = wr;
      bad |= !finite(wr);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// Superset-mask pattern kernels: k_level0_pat / k_level_pat with the row sum
// unrolled over the union of offsets (row_dot_m).  Same rows, same order of
// rounded operations: bit-identical to the table-walking kernels above.
#ifndef SS_MINB
#define SS_MINB 0
#endif
#if SS_MINB > 0
#define SS_LB __launch_bounds__(ROWS_PER_CTA, SS_MINB)
#else
#define SS_LB __launch_bounds__(ROWS_PER_CTA)
#endif
template <typename ID, int NE>
__global__ void SS_LB k_level0_ss(Ctx c) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const SsSmem S = load_ss(c);
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
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int pid_next = i < plim ? row_pattern<ID>(c, i) : 0;
  for (; i < plim; i += stride) {
    const int pid = pid_next;
    {
      const double* pf[3] = {c.x, P0, R0};
      prefetch_next<3>(c, i, stride, pf);
    }
    if (i + stride < plim) pid_next = row_pattern<ID>(c, i + stride);
    double acc[3];
    const double* xs[3] = {c.x, P0, R0};
    const bool rrow = do_r && i < rlim;
    if (rrow)
      row_dot_m<3, NE>(c, S, pid, i, xs, acc);
    else
      row_dot_m<2, NE>(c, S, pid, i, xs, acc);
    const double p = P0[i];
    if (i < n_own) {
      const double r = R0[i];
      const double t = __dsub_rn(c.b[i], acc[0]);
      tt = fma(t, t, tt);
      rr = fma(r, r, rr);
    }
    const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
    P1[i] = wp;
    bad |= !finite(wp);
    if (rrow) {
      const double wr = recur(acc[2], R0[i], 0.0, th, ga, 0.0, false);
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

template <typename ID, int NE>
__global__ void SS_LB k_level_ss(Ctx c, int l) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const SsSmem S = load_ss(c);
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
  const int64_t plim = lvl_p_rows(c, sigma, l), rlim = lvl_r_rows(c, sigma, l);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int pid_next = i < plim ? row_pattern<ID>(c, i) : 0;
  for (; i < plim; i += stride) {
    const int pid = pid_next;
    {
      const double* pf[2] = {Pl, Rl};
      prefetch_next<2>(c, i, stride, pf);
    }
    if (i + stride < plim) pid_next = row_pattern<ID>(c, i + stride);
    double acc[2];
    const double* xs[2] = {Pl, Rl};
    const bool rrow = do_r && i < rlim;
    if (rrow)
      row_dot_m<2, NE>(c, S, pid, i, xs, acc);
    else
      row_dot_m<1, NE>(c, S, pid, i, xs, acc);
    const double wp = recur(acc[0], Pl[i], use_mu ? Pm[i] : 0.0, th, ga, mu, use_mu);
    Pn[i] = wp;
    bad |= !finite(wp);
    if (rrow) {
      const double wr = recur(acc[1], Rl[i], use_mu ? Rm[i] : 0.0, th, ga, mu, use_mu);
      Rn[i] = wr;
      bad |= !finite(wr);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// ---------------------------------------------------------------------------
// Plane-march pattern kernels (Ctx::zm_*).  The union of offsets is
// [-S, ..., 0, ..., +S] (a stencil: S is the plane stride).  A work item is
// 256 consecutive columns c (c = row mod S) x zm_zc consecutive steps; each
// thread walks its column, keeping x[r - S], x[r], x[r + S] in registers, so
// per row and vector one coalesced load (the plane ahead) replaces three
// gathers; the other slots are gathered as in row_dot_m.  The adds run over
// the slots in union order = stored order, absent slots adding +0.0 (exact,
// see row_dot_m): bit-identical to the other level kernels.
// plane table of a row-partitioned march (Ctx::zm_base) in dynamic shared
// memory after the pattern table (load_ss); nullptr: plane z starts at z * S.
// Callers run load_ss first (its barrier also covers this copy: the copy is
// issued before it by the same threads -- see k_level0_zm / k_level_zm).
__device__ __forceinline__ int* zm_plane_smem(const Ctx& c) {
  extern __shared__ __align__(16) double psm[];
  return reinterpret_cast<int*>(reinterpret_cast<char*>(psm) + ss_smem_bytes_dev(c.pat_np));
}
__device__ __forceinline__ void zm_plane_copy(const Ctx& c) {
  if (!c.zm_base) return;
  int* sb = zm_plane_smem(c);
  for (int i = threadIdx.x; i < c.zm_np; i += blockDim.x) sb[i] = __ldg(c.zm_base + i);
}
__device__ __forceinline__ const int* zm_plane_table(const Ctx& c) {
  return c.zm_base ? zm_plane_smem(c) : nullptr;
}

#ifndef ZM_L2PF  // per-thread L2 prefetch of the plane ZM_L2PF steps ahead (c5w: 1 -> +1.5 %, 2 -> -1.3 %, 3 -> -0.6 %, 4-8: 0)
#define ZM_L2PF 2
#endif
#ifndef ZM_PIPE  // plane-ahead loads one step early (measured slower: registers)
#define ZM_PIPE 0
#endif
template <bool UNIT>
__device__ __forceinline__ double recur_t(double ay, double y, double y2, double th, double ga,
                                          double mu, bool use_mu) {
  double w = __dsub_rn(ay, __dmul_rn(th, y));
  if (use_mu) w = __dsub_rn(w, __dmul_rn(mu, y2));
  return UNIT ? w : __ddiv_rn(w, ga);
}

// one column of one work item.  NV input vectors xs[0..NV) (level 0: x, P0, R0
// with NV = 3; else P_l, R_l with NV = 2, or P_l alone with NV = 1).
// MODE: ZM_LEVEL level l >= 1 (NV = 1 or 2 inputs, each with an output);
// ZM_L0 fused level 0 (x, P0, R0 in; P1, R1 out; ||b - A x||^2 and ||r||^2
// partials)
// RK: recurrence kind, bit 0 = non-unit gamma (IEEE division), bit 1 = mu != 0
// (two-back term) -- compile-time, so the Newton levels carry neither
enum { ZM_LEVEL = 0, ZM_L0 = 1 };
template <typename ID, int NE, int NV, int MODE, int RK, bool TAB>
__device__ __forceinline__ void zm_column(const Ctx& c, const SsSmem& T, const int* __restrict__ sbase,
                                          int col, int z0, int z1,
                                          const double* const* __restrict__ xs,
                                          const double* const* __restrict__ ym,
                                          double* const* __restrict__ yo, double th, double ga,
                                          double mu, bool use_mu, int plim, int rlim, int& bad,
                                          double& tt, double& rr) {
  constexpr int KC = NE / 2;
  constexpr bool UNIT = (RK & 1) == 0, MU = (RK & 2) != 0 && MODE == ZM_LEVEL;
  constexpr int NO = MODE == ZM_L0 ? NV - 1 : NV;  // output vectors
  constexpr int Q0 = MODE == ZM_L0 ? 1 : 0;  // first input vector with an output
  constexpr bool TT = MODE == ZM_L0;  // ||b - A x||^2 (acc[0])
  constexpr bool RR = MODE == ZM_L0;  // ||r||^2 (the last input)
  // 32-bit row indices (plan.cu enables the march only for ld + S < 2^31).
  // Plane z of the walk starts at local row sbase[z] (a row-partitioned plan:
  // owned planes, then ghost planes by depth) or z * S (sbase == nullptr).
  // Vectors hold ld >= local rows entries.
  const int S = (int)c.zm_S, n = (int)(c.ld < INT32_MAX ? c.ld : INT32_MAX), n_own = (int)c.n_own;
  const int np = c.zm_np;
  if (z1 > np) z1 = np;
  auto row_of = [&](int z) { return (TAB ? sbase[z] : z * S) + col; };
  int r = row_of(z0);
  double pv[NV], cu[NV];
  {
    const int rp = z0 > 0 ? row_of(z0 - 1) : -1;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      pv[q] = rp >= 0 && rp < n ? __ldg(xs[q] + rp) : 0.0;
      cu[q] = r < n ? __ldg(xs[q] + r) : 0.0;
    }
  }
  // row ids two steps ahead and the row of the next plane one step ahead
  const ID* pidp = reinterpret_cast<const ID*>(c.pid);
  int r1 = z0 + 1 < np ? row_of(z0 + 1) : n;  // row of plane z + 1
  int pid_cur = r < plim ? (int)__ldg(pidp + r) : 0;
  int pid_n1 = (z0 + 1 < z1 && r1 < plim) ? (int)__ldg(pidp + r1) : 0;
  for (int z = z0; z < z1; ++z) {
    const int pid = pid_cur;
    SSCG_CHECK(pid < c.pat_np);
    const int r2 = z + 2 < np ? row_of(z + 2) : n;
    const int pid_n2 = (z + 2 < z1 && r2 < plim) ? (int)__ldg(pidp + r2) : 0;
    double nx[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) nx[q] = r1 < n ? __ldg(xs[q] + r1) : 0.0;
#if ZM_L2PF > 0
    if (z + ZM_L2PF < np) {
      const int rf = row_of(z + ZM_L2PF);
      if (rf < n) {
#pragma unroll
        for (int q = 0; q < NV; ++q) asm volatile("prefetch.global.L2 [%0];" ::"l"(xs[q] + rf));
        if (TT && rf < n_own) asm volatile("prefetch.global.L2 [%0];" ::"l"(c.b + rf));
      }
    }
#endif
    if (r < plim) {
      const bool rrow = r < rlim;  // the last vector (R) is produced on this row
      // Absent slots carry the value 0.0 in the pattern table; they read the
      // row's own entry (offset 0: always in range) or the register slot as
      // is.  Every input a live level reads is finite (a non-finite column
      // ends the solve: basis.py:220, adaptive.py:146), so an absent slot adds
      // 0.0 * x = +-0.0, which leaves any partial sum csr_matvec can hold
      // unchanged (a sum that starts at +0.0 is never -0.0 under
      // round-to-nearest): bit-identical to skipping the slot.
      double xb[NV][NE];
      const int4 eo = T.eoff[pid];  // middle-slot offsets of this row (0: absent)
#pragma unroll
      for (int k = 1; k < NE - 1; ++k) {
        if (k == KC) continue;
        const int o = NE == 7 ? (k == 1 ? eo.x : k == 2 ? eo.y : k == 4 ? eo.z : eo.w)
                              : (k == 1 ? eo.x : eo.y);
#pragma unroll
        for (int q = 0; q < NV; ++q) xb[q][k] = __ldg(xs[q] + (r + o));
      }
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        xb[q][0] = pv[q];
        xb[q][KC] = cu[q];
        xb[q][NE - 1] = nx[q];
      }
      const double2* v2 = reinterpret_cast<const double2*>(T.val + pid * SS_MAX_NE);
      double acc[NV];
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
      if (TT && r < n_own) {
        const double t = __dsub_rn(c.b[r], acc[0]);
        tt = fma(t, t, tt);
      }
      if (RR && r < n_own) rr = fma(cu[NV - 1], cu[NV - 1], rr);
#pragma unroll
      for (int q = 0; q < NO; ++q) {
        if (q == NO - 1 && NO > 1 && !rrow) break;
        const double y2 = MU ? ym[q][r] : 0.0;
        const double w = recur_t<UNIT>(acc[Q0 + q], cu[Q0 + q], y2, th, ga, mu, MU);
        SSCG_CHECK(r >= 0 && r < c.ld);
        yo[q][r] = w;
        bad |= !finite(w);
      }
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      pv[q] = cu[q];
      cu[q] = nx[q];
    }
    pid_cur = pid_n1;
    pid_n1 = pid_n2;
    r = r1;
    r1 = r2;
  }
}

template <typename ID, int NE, int NV, int MODE, int RK>
__device__ __forceinline__ void zm_items(const Ctx& c, int lvl, const SsSmem& T,
                                         const double* const* xs,
                                         const double* const* ym, double* const* yo, double th,
                                         double ga, double mu, bool use_mu, int64_t plim,
                                         int64_t rlim, int& bad, double& tt, double& rr) {
  // level 0 and the residual use fixed stripes with their own item size
  // (zm_zc0: whole rounds of items over the grid), levels >= 1 zm_zc
  const bool l0 = MODE != ZM_LEVEL;
  const int items = (int)(l0 ? c.zm_items0 : c.zm_items), ncb = c.zm_ncb;
  const int zcs = l0 ? c.zm_zc0 : c.zm_zc, S = (int)c.zm_S;
  const int* sbase = zm_plane_table(c);
  // levels >= 1 with Ctx::zm_ctr: the CTA claims items from a per-level
  // counter instead of a fixed stripe, so a CTA that started late (its SM
  // slot held by a Leja-point kernel of the side branch) takes fewer items
  // instead of delaying the whole level.  The row arithmetic is unchanged.
  // (only while the Leja chain of this block runs: st->leja_on; a Chebyshev
  // or monomial basis has no side branch and keeps the fixed stripes)
  const bool dyn = MODE == ZM_LEVEL && c.zm_ctr != nullptr && c.st->leja_on;
  __shared__ int s_claim;
  unsigned* ctr = dyn ? c.zm_ctr + 2 * lvl : nullptr;
  int it = blockIdx.x;
  if (dyn) {
    if (threadIdx.x == 0) s_claim = (int)atomicAdd(ctr, 1u);
    __syncthreads();
    it = s_claim;
  }
  for (; it < items;) {
    const int cb = it % ncb, zc = it / ncb;
    int col;
    if (c.zm_o > 0) {
      // 2-D tile of the plane: 32 consecutive columns per warp (x), the 8
      // warps on consecutive lines of stride zm_o (y), so a row's +-zm_o
      // neighbours are mostly rows another warp of this CTA just loaded (L1)
      const int ntx = c.zm_o >> 5;
      const int ty = (cb / ntx) * (ROWS_PER_CTA / 32) + (threadIdx.x >> 5);
      col = ty * c.zm_o + (cb % ntx) * 32 + (threadIdx.x & 31);
      if (ty >= S / c.zm_o) goto next_item;
    } else {
      col = cb * ROWS_PER_CTA + threadIdx.x;
    }
    if (col >= S) goto next_item;
    {
      const int z0 = zc * zcs;
      if (sbase)  // plane table (partitioned) or arithmetic planes, a compile-time choice
        zm_column<ID, NE, NV, MODE, RK, true>(c, T, sbase, col, z0, z0 + zcs, xs, ym, yo, th, ga,
                                              mu, use_mu, (int)plim, (int)rlim, bad, tt, rr);
      else
        zm_column<ID, NE, NV, MODE, RK, false>(c, T, sbase, col, z0, z0 + zcs, xs, ym, yo, th, ga,
                                               mu, use_mu, (int)plim, (int)rlim, bad, tt, rr);
    }
  next_item:
    if (dyn) {
      __syncthreads();  // every thread has read s_claim
      if (threadIdx.x == 0) s_claim = (int)atomicAdd(ctr, 1u);
      __syncthreads();
      it = s_claim;
    } else {
      it += gridDim.x;
    }
  }
  if (dyn && threadIdx.x == 0 && atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
    atomicExch(ctr, 0u);  // the last CTA out resets the counters for the next launch
    atomicExch(ctr + 1, 0u);
  }
}

#ifndef ZM0_MINB  // 64 registers, no spills: 4 CTAs/SM (1.52 vs 1.58 ms/outer at 3)
#define ZM0_MINB 4
#endif
template <typename ID, int NE>
__global__ void __launch_bounds__(ROWS_PER_CTA, ZM0_MINB) k_level0_zm(Ctx c, ZmPtrs zp) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  zm_plane_copy(c);
  const SsSmem T = load_ss(c);
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  double* yo[2] = {zp.yo[0], zp.yo[1]};
  const double* xs[3] = {zp.xs[0], zp.xs[1], zp.xs[2]};
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int64_t plim = lvl_p_rows(c, sigma, 0), rlim = do_r ? lvl_r_rows(c, sigma, 0) : 0;
  if (ga == 1.0) {
    zm_items<ID, NE, 3, ZM_L0, 0>(c, 0, T, xs, nullptr, yo, th, ga, 0.0, false, plim, rlim, bad, tt, rr);
  } else {
    zm_items<ID, NE, 3, ZM_L0, 1>(c, 0, T, xs, nullptr, yo, th, ga, 0.0, false, plim, rlim, bad, tt, rr);
  }
  rr = block_sum<ROWS_PER_CTA>(rr, sm);
  tt = block_sum<ROWS_PER_CTA>(tt, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = tt;
    c.part_r[blockIdx.x] = rr;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

#ifndef ZM_MINB
#define ZM_MINB 4
#endif
template <typename ID, int NE>
__global__ void __launch_bounds__(ROWS_PER_CTA, ZM_MINB) k_level_zm(Ctx c, int l, ZmPtrs zp) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  zm_plane_copy(c);
  const SsSmem T = load_ss(c);
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const double* xs[2] = {zp.xs[0], zp.xs[1]};
  const double* ym[2] = {zp.ym[0], zp.ym[1]};
  double* yo[2] = {zp.yo[0], zp.yo[1]};
  int bad = 0;
  double tt = 0.0, rr = 0.0;
  const int64_t plim = lvl_p_rows(c, sigma, l), rlim = lvl_r_rows(c, sigma, l);
  const int rk = (ga == 1.0 ? 0 : 1) | (use_mu ? 2 : 0);
#define ZM_RK(NV, RL)                                                                          \
  switch (rk) {                                                                                \
    case 0: zm_items<ID, NE, NV, ZM_LEVEL, 0>(c, l, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad, tt, rr); break; \
    case 1: zm_items<ID, NE, NV, ZM_LEVEL, 1>(c, l, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad, tt, rr); break; \
    case 2: zm_items<ID, NE, NV, ZM_LEVEL, 2>(c, l, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad, tt, rr); break; \
    default: zm_items<ID, NE, NV, ZM_LEVEL, 3>(c, l, T, xs, ym, yo, th, ga, mu, use_mu, plim, RL, bad, tt, rr); break; \
  }
  if (do_r) {
    ZM_RK(2, rlim)
  } else {
    ZM_RK(1, plim)
  }
#undef ZM_RK
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&c.st->breakdown, 1);
}

// ---------------------------------------------------------------------------
// Value-stream stencil kernels (Ctx::vs_*): operators with a stencil's column
// structure but row-varying values (c4: 27-point variable coefficients) do not
// compress to patterns; here the column structure is the union of offsets
// (kernel parameters) and the values stream slot-major, coalesced, 8 bytes per
// slot and row -- no column indices, no row pointers (12 nnz + 4 n bytes of
// CSR become 8 ne n).  One row per thread, slots in union order = stored order,
// in chunks of VS_CHUNK (gathers of a chunk in flight together).  An absent
// slot has value 0.0 and gathers from the clamped index (in range, finite:
// see zm_column): adding 0.0 * x = +-0.0 is exact -- bit-identical to CSR.
#ifndef VS_CHUNK
#define VS_CHUNK 7  // slots per batch of gathers
#endif
// neighbour row of union slot k.  PL (a row-partitioned plan): slot k lies
// vs_dz[k] in {-1, 0, 1} planes away at vs_r[k] rows within the plane; pb[]
// holds the local first rows of the planes below / of / above the row (the
// row's own plane where one is not held -- absent slots only, value 0.0).
// Either way an absent slot reads some in-range row (clamped).
template <bool PL>
__device__ __forceinline__ int vs_nbr(const Ctx& c, int i, int nm1, int k, const int* pb, int pin) {
  if (!PL) return min(max(i + c.vs_off[k], 0), nm1);
  return min(max(pb[c.vs_dz[k] + 1] + pin + c.vs_r[k], 0), nm1);
}

// The value stream is the DRAM stream of these kernels, so each chunk's values
// are requested VS_DEPTH chunks before their use -- across rows too: vq holds
// the next VS_DEPTH chunks (of this row, then of the row this thread handles
// next, inext; < 0: none), a register queue the unrolled loop renames for free.
// PL: the row is row `pin` of local block `blk` (the kernels carry both from
// row to row: one division per thread, not per row).
#ifndef VS_DEPTH
#define VS_DEPTH 1
#endif
#ifndef VS_MINB
#define VS_MINB 4  // CTAs per SM the register allocation must allow (64 registers)
#endif
// (block, row within the block) of a thread's rows i0, i0 + stride, ...
template <bool PL>
struct VsWalk {
  int blk = 0, pin = 0, dblk = 0, dpin = 0, S = 1;
  __device__ __forceinline__ VsWalk(const Ctx& c, int i0, int stride) {
    if (PL) {
      S = (int)c.vs_S;
      blk = i0 / S;
      pin = i0 - blk * S;
      dblk = stride / S;
      dpin = stride - dblk * S;
    }
  }
  __device__ __forceinline__ void next() {
    if (PL) {
      blk += dblk;
      pin += dpin;
      if (pin >= S) {
        pin -= S;
        ++blk;
      }
    }
  }
};

// SYM (Ctx::vs_sym: a bitwise symmetric operator whose union is NE offsets,
// NE odd): only the diagonal's and the upper offsets' planes are stored
// (vs_val[(k - NE/2) * ld + row], k >= NE/2).  The value of a lower offset -o
// at row i is A[i][i - o] = A[i - o][i]: the upper plane of +o at row i - o --
// the same coalesced stream, o rows earlier (0.0 where i - o < 0: no such
// neighbour).  An element is read as an upper value by row i and as a lower one
// by row i + o, at most vs_off[NE - 1] rows later: the second read comes from
// L2, the DRAM stream is (NE + 1) / 2 planes instead of NE.
template <int NE, bool SYM = false>
__device__ __forceinline__ void vs_request(const Ctx& c, int i, int chunk, double (&v)[VS_CHUNK]) {
  if (!SYM) {
    const double* vp = c.vs_val + i + (int64_t)(chunk * VS_CHUNK) * c.ld;
#pragma unroll
    for (int kk = 0; kk < VS_CHUNK; ++kk)
      if (chunk * VS_CHUNK + kk < NE) v[kk] = __ldg(vp + (int64_t)kk * c.ld);
  } else {
    constexpr int MID = NE / 2;
#pragma unroll
    for (int kk = 0; kk < VS_CHUNK; ++kk) {
      const int k = chunk * VS_CHUNK + kk;
      if (k >= NE) continue;
      if (k >= MID) {
        v[kk] = __ldg(c.vs_val + i + (int64_t)(k - MID) * c.ld);
      } else {
        const int j = i + c.vs_off[k];  // the row that stores this entry
        v[kk] = j >= 0 ? __ldg(c.vs_val + j + (int64_t)(NE - 1 - k - MID) * c.ld) : 0.0;
      }
    }
  }
}
// the first row's first VS_DEPTH chunks
template <int NE, bool SYM = false>
__device__ __forceinline__ void vs_first(const Ctx& c, int i, double (&vq)[VS_DEPTH][VS_CHUNK]) {
#pragma unroll
  constexpr int NCH = (NE + VS_CHUNK - 1) / VS_CHUNK;
#pragma unroll
  for (int d = 0; d < (VS_DEPTH < NCH ? VS_DEPTH : NCH); ++d) vs_request<NE, SYM>(c, i, d, vq[d]);
}

template <int NV, int NE, bool PL = false, bool SYM = false>
__device__ __forceinline__ void vs_row(const Ctx& c, int i, int nm1,
                                       const double* const* __restrict__ xs, double* acc,
                                       double (&vq)[VS_DEPTH][VS_CHUNK], int inext, int blk = 0,
                                       int pin = 0) {
  constexpr int NCH = (NE + VS_CHUNK - 1) / VS_CHUNK;
  constexpr int D = VS_DEPTH < NCH ? VS_DEPTH : NCH;  // the queue reaches at most one row ahead
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  int pb[3] = {0, 0, 0};
  if (PL) {
    pb[0] = __ldg(c.vs_below + blk);
    pb[1] = i - pin;
    pb[2] = __ldg(c.vs_above + blk);
  }
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch) {
    const int k0 = ch * VS_CHUNK;
    double v[VS_CHUNK], xb[NV][VS_CHUNK];
#pragma unroll
    for (int kk = 0; kk < VS_CHUNK; ++kk) v[kk] = vq[0][kk];
#pragma unroll
    for (int d = 0; d + 1 < D; ++d)
#pragma unroll
      for (int kk = 0; kk < VS_CHUNK; ++kk) vq[d][kk] = vq[d + 1][kk];
    if (ch + D < NCH)
      vs_request<NE, SYM>(c, i, ch + D, vq[D - 1]);
    else if (inext >= 0)
      vs_request<NE, SYM>(c, inext, ch + D - NCH, vq[D - 1]);
#pragma unroll
    for (int kk = 0; kk < VS_CHUNK; ++kk) {
      const int k = k0 + kk;
      if (k < NE) {
        const int j = vs_nbr<PL>(c, i, nm1, k, pb, pin);
        SSCG_CHECK(j >= 0 && j < c.ld);
#pragma unroll
        for (int q = 0; q < NV; ++q) xb[q][kk] = __ldg(xs[q] + j);
      }
    }
#pragma unroll
    for (int kk = 0; kk < VS_CHUNK; ++kk) {
      if (k0 + kk < NE) {
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(v[kk], xb[q][kk]));
      }
    }
  }
}

template <int NE, bool PL, bool SYM = false>
__global__ void __launch_bounds__(ROWS_PER_CTA, VS_MINB) k_level0_vs(Ctx c, ZmPtrs zp) {
  __shared__ double sm[ROWS_PER_CTA / 32];
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[0], ga = st->prm.ga[0];
  const bool do_r = sbar >= 2;
  const double* xs[3] = {zp.xs[0], zp.xs[1], zp.xs[2]};
  double tt = 0.0, rr = 0.0;
  int bad = 0;
  const int n_own = (int)c.n_own, plim = (int)lvl_p_rows(c, sigma, 0);
  const int rlim = do_r ? (int)lvl_r_rows(c, sigma, 0) : 0;
  const int nm1 = (int)(PL ? c.lvl_rows[SMAX] : c.n) - 1;
  const int stride = gridDim.x * blockDim.x;
  double vn[VS_DEPTH][VS_CHUNK];
  if ((int)(blockIdx.x * blockDim.x + threadIdx.x) < plim)
    vs_first<NE, SYM>(c, blockIdx.x * blockDim.x + threadIdx.x, vn);
  VsWalk<PL> w(c, blockIdx.x * blockDim.x + threadIdx.x, stride);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < plim; i += stride, w.next()) {
    double acc[3];
    vs_row<3, NE, PL, SYM>(c, i, nm1, xs, acc, vn, i + stride < plim ? i + stride : -1, w.blk, w.pin);
    const double p = xs[1][i], r = xs[2][i];
    if (i < n_own) {
      const double t = __dsub_rn(c.b[i], acc[0]);
      tt = fma(t, t, tt);
      rr = fma(r, r, rr);
    }
    const double wp = recur(acc[1], p, 0.0, th, ga, 0.0, false);
    zp.yo[0][i] = wp;
    bad |= !finite(wp);
    if (i < rlim) {
      const double wr = recur(acc[2], r, 0.0, th, ga, 0.0, false);
      zp.yo[1][i] = wr;
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

template <int NE, bool PL, bool SYM = false>
__global__ void __launch_bounds__(ROWS_PER_CTA, VS_MINB) k_level_vs(Ctx c, int l, ZmPtrs zp) {
  const SolverState* st = c.st;
  if (st->done) return;
  const int sbar = st->s_bar;
  if (l >= sbar) return;
  const int sigma = c.cfg->sigma;
  const double th = st->prm.th[l], ga = st->prm.ga[l], mu = st->prm.mu[l - 1];
  const bool use_mu = !(mu == 0.0);  // basis.py:217 `if mu != 0.0` (NaN counts)
  const bool do_r = l < sbar - 1;
  const int plim = (int)lvl_p_rows(c, sigma, l), rlim = (int)lvl_r_rows(c, sigma, l);
  const int nm1 = (int)(PL ? c.lvl_rows[SMAX] : c.n) - 1;
  const int stride = gridDim.x * blockDim.x;
  int bad = 0;
  const double* xs[2] = {zp.xs[0], zp.xs[1]};
  double vn[VS_DEPTH][VS_CHUNK];
  if ((int)(blockIdx.x * blockDim.x + threadIdx.x) < plim)
    vs_first<NE, SYM>(c, blockIdx.x * blockDim.x + threadIdx.x, vn);
  VsWalk<PL> w(c, blockIdx.x * blockDim.x + threadIdx.x, stride);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < plim; i += stride, w.next()) {
    double acc[2];
    const bool rrow = do_r && i < rlim;
    const int inext = i + stride < plim ? i + stride : -1;
    if (rrow)
      vs_row<2, NE, PL, SYM>(c, i, nm1, xs, acc, vn, inext, w.blk, w.pin);
    else
      vs_row<1, NE, PL, SYM>(c, i, nm1, xs, acc, vn, inext, w.blk, w.pin);
    const double wp = recur(acc[0], xs[0][i], use_mu ? zp.ym[0][i] : 0.0, th, ga, mu, use_mu);
    zp.yo[0][i] = wp;
    bad |= !finite(wp);
    if (rrow) {
      const double wr = recur(acc[1], xs[1][i], use_mu ? zp.ym[1][i] : 0.0, th, ga, mu, use_mu);
      zp.yo[1][i] = wr;
      bad |= !finite(wr);
    }
  }
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
size_t pattern_smem_bytes(int np, int ne) {
  return (size_t)ne * 12 + (size_t)(np + 1) * 4;
}

void pattern_prepare() {
  const int bytes = 48 * 1024;
  cudaFuncSetAttribute(k_level0_pat<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_level0_pat<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_level_pat<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_level_pat<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

size_t ss_smem_bytes(int np) { return ss_smem_bytes_dev(np); }

int ss_ne_bucket(int ne) { return ne <= 3 ? 3 : ne <= 5 ? 5 : ne <= 7 ? 7 : 8; }

template <typename ID, int NE>
void ss_occ(size_t bytes, int* a, int* b) {
  const int lim = 48 * 1024;
  cudaFuncSetAttribute(k_level0_ss<ID, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(k_level_ss<ID, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(a, k_level0_ss<ID, NE>, ROWS_PER_CTA, bytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(b, k_level_ss<ID, NE>, ROWS_PER_CTA, bytes);
}

template <typename ID, int NE>
void zm_occ(size_t bytes, int* a, int* b) {
  const int lim = 48 * 1024;
  cudaFuncSetAttribute(k_level0_zm<ID, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaFuncSetAttribute(k_level_zm<ID, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(a, k_level0_zm<ID, NE>, ROWS_PER_CTA, bytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(b, k_level_zm<ID, NE>, ROWS_PER_CTA, bytes);
}

// plane-march kernels for a symmetric union of 3, 5 or 7 offsets
int zm_ctas_per_sm(int np, int ne, int pid_bytes, int* out2) {
  int a = 0, b = 0;
  const size_t bytes = ss_smem_bytes_dev(np);
  if (ne != 3 && ne != 5 && ne != 7) return 0;
  if (pid_bytes == 1) {
    if (ne == 3) zm_occ<uint8_t, 3>(bytes, &a, &b);
    else if (ne == 5) zm_occ<uint8_t, 5>(bytes, &a, &b);
    else zm_occ<uint8_t, 7>(bytes, &a, &b);
  } else {
    if (ne == 3) zm_occ<uint16_t, 3>(bytes, &a, &b);
    else if (ne == 5) zm_occ<uint16_t, 5>(bytes, &a, &b);
    else zm_occ<uint16_t, 7>(bytes, &a, &b);
  }
  out2[0] = a;
  out2[1] = b;
  return a < b ? a : b;
}

// value-stream kernels (plain or plane-table form): CTAs per SM of level 0
// and levels >= 1
int vs_ctas_per_sm(int ne, bool pl, int* out2) {
  const int nb = ne <= 9 ? 9 : ne <= 18 ? 18 : ne <= 27 ? 27 : 32;
  int a = 0, b = 0;
#define VS_OCC(NE)                                                                              \
  if (pl) {                                                                                     \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_level0_vs<NE, true>, ROWS_PER_CTA, 0);  \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_level_vs<NE, true>, ROWS_PER_CTA, 0);   \
  } else {                                                                                      \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_level0_vs<NE, false>, ROWS_PER_CTA, 0); \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_level_vs<NE, false>, ROWS_PER_CTA, 0);  \
  }
  if (nb == 9) { VS_OCC(9) } else if (nb == 18) { VS_OCC(18) } else if (nb == 27) { VS_OCC(27) } else { VS_OCC(32) }
#undef VS_OCC
  out2[0] = a;
  out2[1] = b;
  return a < b ? a : b;
}

int ss_ctas_per_sm(int np, int ne, int pid_bytes, int* out2) {
  int a = 0, b = 0;
  const size_t bytes = ss_smem_bytes_dev(np);
  const int nb = ss_ne_bucket(ne);
  if (pid_bytes == 1) {
    if (nb == 3) ss_occ<uint8_t, 3>(bytes, &a, &b);
    else if (nb == 5) ss_occ<uint8_t, 5>(bytes, &a, &b);
    else if (nb == 7) ss_occ<uint8_t, 7>(bytes, &a, &b);
    else ss_occ<uint8_t, 8>(bytes, &a, &b);
  } else {
    if (nb == 3) ss_occ<uint16_t, 3>(bytes, &a, &b);
    else if (nb == 5) ss_occ<uint16_t, 5>(bytes, &a, &b);
    else if (nb == 7) ss_occ<uint16_t, 7>(bytes, &a, &b);
    else ss_occ<uint16_t, 8>(bytes, &a, &b);
  }
  out2[0] = a;
  out2[1] = b;
  return a < b ? a : b;
}

// level 0 (the partial-sum kernel) and levels >= 1: out[0], out[1]
int pattern_ctas_per_sm(int np, int ne, int pid_bytes, int* out2) {
  int a = 0, b = 0;
  const size_t bytes = pattern_smem_bytes(np, ne);
  if (pid_bytes == 1) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_level0_pat<uint8_t>, ROWS_PER_CTA, bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_level_pat<uint8_t>, ROWS_PER_CTA, bytes);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_level0_pat<uint16_t>, ROWS_PER_CTA, bytes);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_level_pat<uint16_t>, ROWS_PER_CTA, bytes);
  }
  out2[0] = a;
  out2[1] = b;
  return a < b ? a : b;
}

void launch_level(const Ctx& c, int level, int sigma, cudaStream_t s) {
  if (c.vs_ne > 0) {
    const ZmPtrs zp = zm_ptrs(c, level, sigma);
    const int ne = c.vs_ne <= 9 ? 9 : c.vs_ne <= 18 ? 18 : c.vs_ne <= 27 ? 27 : 32;
#define VS_LAUNCH(NE)                                                        \
  if (level == 0 && c.vs_S)                                                  \
    k_level0_vs<NE, true><<<c.red_n, ROWS_PER_CTA, 0, s>>>(c, zp);           \
  else if (level == 0)                                                       \
    k_level0_vs<NE, false><<<c.red_n, ROWS_PER_CTA, 0, s>>>(c, zp);          \
  else if (c.vs_S)                                                           \
    k_level_vs<NE, true><<<c.pat_grid, ROWS_PER_CTA, 0, s>>>(c, level, zp);  \
  else                                                                       \
    k_level_vs<NE, false><<<c.pat_grid, ROWS_PER_CTA, 0, s>>>(c, level, zp);
#define VS_LAUNCH_SYM(NE)                                                          \
  if (level == 0)                                                                  \
    k_level0_vs<NE, false, true><<<c.red_n, ROWS_PER_CTA, 0, s>>>(c, zp);          \
  else                                                                             \
    k_level_vs<NE, false, true><<<c.pat_grid, ROWS_PER_CTA, 0, s>>>(c, level, zp);
    if (c.vs_sym && !c.vs_S && (c.vs_ne == 9 || c.vs_ne == 27)) {
      if (c.vs_ne == 9) {
        VS_LAUNCH_SYM(9)
      } else {
        VS_LAUNCH_SYM(27)
      }
      return;
    }
#undef VS_LAUNCH_SYM
    switch (ne) {
      case 9: VS_LAUNCH(9) break;
      case 18: VS_LAUNCH(18) break;
      case 27: VS_LAUNCH(27) break;
      default: VS_LAUNCH(32) break;
    }
#undef VS_LAUNCH
    return;
  }
  if (c.tm) {  // the TMA plane march (tmarch.cu)
    launch_level_tm(c, level, sigma, s);
    return;
  }
  if (c.pid && c.ss_ne > 0 && c.zm_S > 0) {
    const size_t bytes = ss_smem_bytes_dev(c.pat_np) + (c.zm_base ? 4 * (size_t)c.zm_np : 0);
    const ZmPtrs zp = zm_ptrs(c, level, sigma);
#define ZM_LAUNCH(ID, NE)                                                      \
  if (level == 0)                                                              \
    k_level0_zm<ID, NE><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c, zp);           \
  else                                                                         \
    k_level_zm<ID, NE><<<c.pat_grid, ROWS_PER_CTA, bytes, s>>>(c, level, zp);
#define ZM_NE_SWITCH(ID)                   \
  switch (c.ss_ne) {                       \
    case 3: ZM_LAUNCH(ID, 3) break;        \
    case 5: ZM_LAUNCH(ID, 5) break;        \
    default: ZM_LAUNCH(ID, 7) break;       \
  }
    if (c.pid_bytes == 1) {
      ZM_NE_SWITCH(uint8_t)
    } else {
      ZM_NE_SWITCH(uint16_t)
    }
    return;
  }
  if (c.pid && c.ss_ne > 0) {
    const size_t bytes = ss_smem_bytes_dev(c.pat_np);
    const int ne = ss_ne_bucket(c.ss_ne);
#define SS_LAUNCH(ID, NE)                                                      \
  if (level == 0)                                                              \
    k_level0_ss<ID, NE><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c);               \
  else                                                                         \
    k_level_ss<ID, NE><<<c.pat_grid, ROWS_PER_CTA, bytes, s>>>(c, level);
#define SS_NE_SWITCH(ID)                   \
  switch (ne) {                            \
    case 3: SS_LAUNCH(ID, 3) break;        \
    case 5: SS_LAUNCH(ID, 5) break;        \
    case 7: SS_LAUNCH(ID, 7) break;        \
    default: SS_LAUNCH(ID, 8) break;       \
  }
    if (c.pid_bytes == 1) {
      SS_NE_SWITCH(uint8_t)
    } else {
      SS_NE_SWITCH(uint16_t)
    }
    return;
  }
  if (c.pid) {
    const size_t bytes = pattern_smem_bytes(c.pat_np, c.pat_ne);
    if (c.pid_bytes == 1) {
      if (level == 0)
        k_level0_pat<uint8_t><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c);
      else
        k_level_pat<uint8_t><<<c.pat_grid, ROWS_PER_CTA, bytes, s>>>(c, level);
    } else {
      if (level == 0)
        k_level0_pat<uint16_t><<<c.red_n, ROWS_PER_CTA, bytes, s>>>(c);
      else
        k_level_pat<uint16_t><<<c.pat_grid, ROWS_PER_CTA, bytes, s>>>(c, level);
    }
    return;
  }
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
