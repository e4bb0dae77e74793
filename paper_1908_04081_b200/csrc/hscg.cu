// hscg.cu -- Hestenes-Stiefel CG on the device (classic.py:33-104; SURVEY.md
// 8(f) row 2: the classic-CG baseline the s-step solver is compared with).
//
// One iteration = three row-streaming kernels, each closed by its last CTA
// (fixed-order reduction of the per-CTA partials, so every run gives the same
// bits):
//   k_hs_ap  : ap = A p and p.ap             -> alpha = rr / p.ap (breakdown check)
//   k_hs_xr  : x += alpha p, r -= alpha ap, r.r -> beta, Ritz absorb, alpha/beta log
//   k_hs_pt  : p = r + beta p and the true residual b - A x (||b-Ax||, ||b-Ax-r||)
//              -> the trace row and the loop-top verdict (converged / diverged /
//              stagnated / max_iters) of the next iteration
// The reference's r.r of iteration i+1 is the dot of the same r its iteration i
// already formed, so it is reused, not recomputed.  Vector updates round op by
// op as numpy does (alpha*p, then +); row sums are the CSR / pattern row sums
// of the matrix-powers kernels (csr_matvec order).
//
// Roofline (HBM): ~105 n bytes per iteration (p, ap, x, r, b passes, two
// SpMV-shaped gathers), ids or CSR once per SpMV.
#include <algorithm>

#include "internal.cuh"
#include "ritz.cuh"
#include "rowops.cuh"

namespace {

constexpr int HS_T = ROWS_PER_CTA;  // 256
// red_buf slots (the buffer allreduced on a partitioned plan)
constexpr int HS_RED_BB = 0, HS_RED_RR = 1;                  // start: ||b||^2, r.r
constexpr int HS_RED_PAP = 0, HS_RED_TT = 1, HS_RED_GG = 2;  // after k_hs_ap (3 doubles)
constexpr int HS_RED_RRN = 3;                                // after k_hs_xr (1 double)

// row sums: 0 = CSR (unstaged), 1 = pattern ids uint8, 2 = pattern ids uint16,
// 3 = superset-mask rows with uint8 ids (the union of offsets unrolled: about
// half the instructions of the table walk; same rounded operations)
template <int MODE>
struct RowSum {
  PatSmem T;
  SsSmem S;
  __device__ __forceinline__ void init(const Ctx& c) {
    if (MODE == 3)
      S = load_ss(c);
    else if (MODE != 0)
      T = load_patterns(c);
  }
  __device__ __forceinline__ double dot(const Ctx& c, int64_t i, const double* x) const {
    double acc[1];
    const double* xs[1] = {x};
    if (MODE == 0) {
      row_dot<1>(c.col, c.val, c.rp[i], c.rp[i + 1], xs, acc);
    } else if (MODE == 3) {
      row_dot_m<1, SS_MAX_NE>(c, S, row_pattern<uint8_t>(c, i), i, xs, acc);
    } else {
      const int pid = MODE == 1 ? row_pattern<uint8_t>(c, i) : row_pattern<uint16_t>(c, i);
      row_dot_p<1>(T, T.ptr[pid], T.ptr[pid + 1], (int)i, xs, acc);
    }
    return acc[0];
  }
};

// every CTA writes its partials, the last one to arrive reduces them
__device__ __forceinline__ bool last_cta(int* counter) {
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// fixed-order sum of n partials (thread-strided, then the block tree)
__device__ __forceinline__ double sum_parts(const double* part, int n, double* sm) {
  double v = 0.0;
  for (int j = threadIdx.x; j < n; j += HS_T) v += part[j];
  return block_sum<HS_T>(v, sm);  // thread 0
}

__device__ __forceinline__ double* hs_log(const Ctx& c, int64_t it) {
  return it < c.cfg->cap_iters ? c.it_log + it * SSCG_IT_N : nullptr;
}

// loop top of classic.py:58-72 for iteration i: the verdict, a pure function
// of the state and the loop-top residuals (every CTA of k_hs_xr evaluates it
// and takes the same branch; only the last CTA writes best / status).
// Production mode (PROD) steers by the updated residual: convergence when
// ||r|| / ||b|| <= eps*, no stagnation test (the true residual is not formed).
__device__ int hs_verdict(const SolverState* st, const DevConfig& cf, double true_rel,
                          double r_norm, bool prod, bool* new_best) {
  const int i = st->total_iters;
  *new_best = false;
  if ((int64_t)i >= cf.max_iters) return SSCG_EXHAUSTED;  // `while i < max_iters` exits first
  if (true_rel <= cf.eps_star) return SSCG_CONVERGED;
  if (!isfinite(true_rel) || true_rel > 1e5) return SSCG_DIVERGED;
  if (true_rel < st->best) {
    *new_best = true;
    return SSCG_RUNNING;
  }
  if (!prod && i - st->best_iter >= 200 && r_norm <= 0.01 * true_rel * st->nb)
    return SSCG_STAGNATED;
  return SSCG_RUNNING;
}

// x = x0, r = b - A x0, p = r over the owned rows (ghost rows: x from x0; p and
// r arrive with the first halo exchange); partials of ||b||^2 and r.r -> red
template <int MODE>
__global__ void __launch_bounds__(HS_T) k_hs_init(Ctx c, double* P, double* R, const double* x0) {
  __shared__ double sm[HS_T / 32];
  RowSum<MODE> A;
  A.init(c);
  SolverState* st = c.st;
  double bb = 0.0, rr = 0.0;
  const int64_t stride = (int64_t)gridDim.x * HS_T;
  for (int64_t i = (int64_t)blockIdx.x * HS_T + threadIdx.x; i < c.lvl_rows[SMAX]; i += stride) {
    c.x[i] = x0[i];
    if (i >= c.n_own) continue;
    const double bi = c.b[i];
    const double r = __dsub_rn(bi, A.dot(c, i, x0));
    R[i] = r;
    P[i] = r;
    bb = fma(bi, bi, bb);
    rr = fma(r, r, rr);
  }
  bb = block_sum<HS_T>(bb, sm);
  rr = block_sum<HS_T>(rr, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = bb;
    c.part_r[blockIdx.x] = rr;
  }
  if (!last_cta(&st->gram_count)) return;
  bb = sum_parts(c.part_t, gridDim.x, sm);
  rr = sum_parts(c.part_r, gridDim.x, sm);
  if (threadIdx.x == 0) {
    st->gram_count = 0;
    c.red_buf[HS_RED_BB] = bb;
    c.red_buf[HS_RED_RR] = rr;
  }
}

// the reduced ||b||^2 and r.r: the solver state (one thread)
__global__ void k_hs_start(Ctx c) {
  SolverState* st = c.st;
  const DevConfig cf = *c.cfg;
  st->k = 0;
  st->done = 0;
  st->status = SSCG_RUNNING;
  st->total_iters = 0;
  st->total_outer = 0;
  st->n_records = 0;
  st->best = INFINITY;
  st->best_iter = 0;
  st->nb = sqrt(c.red_buf[HS_RED_BB]);
  st->hs_rr = c.red_buf[HS_RED_RR];
  ritz_init(st->rz, cf.c0);
}

// ap = A p over the owned rows and p.ap; TV (reference semantics): also the
// true residual of the current x, tv = b - A x, with ||tv||^2 and ||tv - r||^2
// -- classic.py forms it after each update and classifies with it at the next
// loop top; here both happen one kernel later, on the same x
template <int MODE, bool TV>
__global__ void __launch_bounds__(HS_T) k_hs_ap(Ctx c, const double* P, double* AP, const double* R) {
  __shared__ double sm[HS_T / 32];
  SolverState* st = c.st;
  if (st->done) return;
  RowSum<MODE> A;
  A.init(c);
  double pap = 0.0, tt = 0.0, gg = 0.0;
  const int64_t stride = (int64_t)gridDim.x * HS_T;
  for (int64_t i = (int64_t)blockIdx.x * HS_T + threadIdx.x; i < c.n_own; i += stride) {
    const double ap = A.dot(c, i, P);
    AP[i] = ap;
    pap = fma(P[i], ap, pap);
    if (TV) {
      const double tv = __dsub_rn(c.b[i], A.dot(c, i, c.x));
      const double gv = __dsub_rn(tv, R[i]);
      tt = fma(tv, tv, tt);
      gg = fma(gv, gv, gg);
    }
  }
  pap = block_sum<HS_T>(pap, sm);
  if (TV) {
    tt = block_sum<HS_T>(tt, sm);
    gg = block_sum<HS_T>(gg, sm);
  }
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = pap;
    c.part_r[blockIdx.x] = tt;
    c.part_d[blockIdx.x] = gg;
  }
  if (!last_cta(&st->gram_count)) return;
  pap = sum_parts(c.part_t, gridDim.x, sm);
  tt = TV ? sum_parts(c.part_r, gridDim.x, sm) : 0.0;
  gg = TV ? sum_parts(c.part_d, gridDim.x, sm) : 0.0;
  if (threadIdx.x == 0) {
    st->gram_count = 0;
    c.red_buf[HS_RED_PAP] = pap;
    c.red_buf[HS_RED_TT] = tt;
    c.red_buf[HS_RED_GG] = gg;
  }
}

// loop top (the previous iteration's trace row, the verdict), then alpha =
// rr / p.ap (breakdown check, classic.py:77-79), x += alpha p, r -= alpha ap
// and the new r.r partial -> red
__global__ void __launch_bounds__(HS_T) k_hs_xr(Ctx c, const double* P, const double* AP,
                                                double* R, int prod) {
  __shared__ double sm[HS_T / 32];
  SolverState* st = c.st;
  if (st->done) return;
  const DevConfig cf = *c.cfg;
  const double nb = st->nb;
  const double r_norm = sqrt(st->hs_rr);
  const double true_rel = prod ? r_norm / nb : sqrt(c.red_buf[HS_RED_TT]) / nb;
  bool new_best;
  int out = hs_verdict(st, cf, true_rel, r_norm, prod != 0, &new_best);
  const double pap = c.red_buf[HS_RED_PAP];
  if (out == SSCG_RUNNING && (pap <= 0.0 || !isfinite(pap))) out = SSCG_DIVERGED;
  double rr = 0.0;
  if (out == SSCG_RUNNING) {
    const double alpha = st->hs_rr / pap;
    // two rows per thread and step (16-byte accesses; the columns are 16-byte
    // aligned), two steps in flight: a pure stream of 48 bytes per row
    const int64_t n2 = c.n_own & ~(int64_t)1;
    const int64_t stride = (int64_t)gridDim.x * HS_T * 2;
#pragma unroll 2
    for (int64_t i = ((int64_t)blockIdx.x * HS_T + threadIdx.x) * 2; i < n2; i += stride) {
      double2 xv = *reinterpret_cast<const double2*>(c.x + i);
      const double2 pv = *reinterpret_cast<const double2*>(P + i);
      double2 rv = *reinterpret_cast<const double2*>(R + i);
      const double2 av = *reinterpret_cast<const double2*>(AP + i);
      xv.x = __dadd_rn(xv.x, __dmul_rn(alpha, pv.x));  // q = alpha*p; x = x + q
      xv.y = __dadd_rn(xv.y, __dmul_rn(alpha, pv.y));
      rv.x = __dsub_rn(rv.x, __dmul_rn(alpha, av.x));
      rv.y = __dsub_rn(rv.y, __dmul_rn(alpha, av.y));
      *reinterpret_cast<double2*>(c.x + i) = xv;
      *reinterpret_cast<double2*>(R + i) = rv;
      rr = fma(rv.x, rv.x, rr);
      rr = fma(rv.y, rv.y, rr);
    }
    if (n2 < c.n_own && blockIdx.x == 0 && threadIdx.x == 0) {  // odd row count: the last row
      const int64_t i = n2;
      c.x[i] = __dadd_rn(c.x[i], __dmul_rn(alpha, P[i]));
      const double r = __dsub_rn(R[i], __dmul_rn(alpha, AP[i]));
      R[i] = r;
      rr = fma(r, r, rr);
    }
  }
  rr = block_sum<HS_T>(rr, sm);
  if (threadIdx.x == 0) c.part_r[blockIdx.x] = rr;
  if (!last_cta(&st->gram_count)) return;
  rr = sum_parts(c.part_r, gridDim.x, sm);
  if (threadIdx.x == 0) {
    st->gram_count = 0;
    const int it = st->total_iters;
    if (it > 0 && !prod) {  // the previous iteration's row: the true residual of this x
      if (double* row = hs_log(c, it - 1)) {
        row[SSCG_IT_TRUE] = true_rel;
        row[SSCG_IT_GAP] = sqrt(c.red_buf[HS_RED_GG]);
      }
    }
    if (new_best) {
      st->best = true_rel;
      st->best_iter = it;
    }
    if (out != SSCG_RUNNING) {
      st->status = out;
      st->done = 1;
    } else {
      st->hs_alpha = st->hs_rr / pap;
      c.red_buf[HS_RED_RRN] = rr;
    }
  }
}

// beta = rr_new / rr, Ritz absorb, the iteration's log row; p = r + beta p
__global__ void __launch_bounds__(HS_T) k_hs_p(Ctx c, double* P, const double* R) {
  __shared__ double sm[HS_T / 32];
  SolverState* st = c.st;
  if (st->done) return;
  const double rr = c.red_buf[HS_RED_RRN];
  const double beta = rr / st->hs_rr;
  const int64_t n2 = c.n_own & ~(int64_t)1;
  const int64_t stride = (int64_t)gridDim.x * HS_T * 2;
#pragma unroll 2
  for (int64_t i = ((int64_t)blockIdx.x * HS_T + threadIdx.x) * 2; i < n2; i += stride) {
    double2 pv = *reinterpret_cast<const double2*>(P + i);
    const double2 rv = *reinterpret_cast<const double2*>(R + i);
    pv.x = __dadd_rn(rv.x, __dmul_rn(beta, pv.x));
    pv.y = __dadd_rn(rv.y, __dmul_rn(beta, pv.y));
    *reinterpret_cast<double2*>(P + i) = pv;
  }
  if (n2 < c.n_own && blockIdx.x == 0 && threadIdx.x == 0)
    P[n2] = __dadd_rn(R[n2], __dmul_rn(beta, P[n2]));
  if (!last_cta(&st->gram_count)) return;
  if (threadIdx.x == 0) {
    st->gram_count = 0;
    const double alpha = st->hs_alpha;
    const int it = st->total_iters;
    ritz_absorb(st->rz, alpha, beta);  // BreakdownSignal -> state untouched
    if (double* row = hs_log(c, it)) {  // trace.record_iteration (true / gap: next loop top)
      const double nb = st->nb;
      row[SSCG_IT_ALPHA] = alpha;
      row[SSCG_IT_BETA] = beta;
      row[SSCG_IT_UPD] = sqrt(rr) / nb;
      row[SSCG_IT_EST] = sqrt(rr) / nb;
      row[SSCG_IT_XI] = ritz_xi(st->rz);
      row[SSCG_IT_LMIN] = ritz_lmin(st->rz);
      row[SSCG_IT_LMAX] = ritz_lmax(st->rz);
      row[SSCG_IT_PSI] = st->rz.psi;
    }
    st->hs_beta = beta;
    st->hs_rr = rr;
    st->total_iters = it + 1;
    st->total_outer = it + 1;  // trace.mark_outer(1) per iteration
  }
}

// production mode, after the loop: the true residual of the final x for the
// last trace row (one more A x pass; ghost x arrive with the halo before it)
template <int MODE>
__global__ void __launch_bounds__(HS_T) k_hs_final(Ctx c, const double* R) {
  __shared__ double sm[HS_T / 32];
  SolverState* st = c.st;
  RowSum<MODE> A;
  A.init(c);
  double tt = 0.0, gg = 0.0;
  const int64_t stride = (int64_t)gridDim.x * HS_T;
  for (int64_t i = (int64_t)blockIdx.x * HS_T + threadIdx.x; i < c.n_own; i += stride) {
    const double tv = __dsub_rn(c.b[i], A.dot(c, i, c.x));
    const double gv = __dsub_rn(tv, R[i]);
    tt = fma(tv, tv, tt);
    gg = fma(gv, gv, gg);
  }
  tt = block_sum<HS_T>(tt, sm);
  gg = block_sum<HS_T>(gg, sm);
  if (threadIdx.x == 0) {
    c.part_r[blockIdx.x] = tt;
    c.part_d[blockIdx.x] = gg;
  }
  if (!last_cta(&st->gram_count)) return;
  tt = sum_parts(c.part_r, gridDim.x, sm);
  gg = sum_parts(c.part_d, gridDim.x, sm);
  if (threadIdx.x == 0) {
    st->gram_count = 0;
    c.red_buf[HS_RED_TT] = tt;
    c.red_buf[HS_RED_GG] = gg;
  }
}

// the final row's true residual (after k_hs_final and its allreduce)
__global__ void k_hs_final_row(Ctx c) {
  SolverState* st = c.st;
  const int it = st->total_iters;
  if (it < 1) return;
  if (double* row = hs_log(c, it - 1)) {
    row[SSCG_IT_TRUE] = sqrt(c.red_buf[HS_RED_TT]) / st->nb;
    row[SSCG_IT_GAP] = sqrt(c.red_buf[HS_RED_GG]);
  }
}

template <int MODE>
void hs_launch_init(const Ctx& c, double* P, double* R, const double* x0, size_t smem,
                    cudaStream_t s) {
  k_hs_init<MODE><<<c.red_n, HS_T, smem, s>>>(c, P, R, x0);
}
template <int MODE>
void hs_launch_ap(const Ctx& c, const double* P, double* AP, const double* R, bool tv, size_t smem,
                  cudaStream_t s) {
  // as many CTAs as the partial-sum arrays hold (8 per SM): the row sums gather
  // through L1 and want every warp slot, not the level kernels' grid
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((c.n_own + HS_T - 1) / HS_T, RED_BLOCKS));
  if (tv)  // (two row sums per row, 78 registers: one wave of the plan's grid is faster)
    k_hs_ap<MODE, true><<<c.red_n, HS_T, smem, s>>>(c, P, AP, R);
  else
    k_hs_ap<MODE, false><<<grid, HS_T, smem, s>>>(c, P, AP, R);
}
template <int MODE>
void hs_launch_final(const Ctx& c, const double* R, size_t smem, cudaStream_t s) {
  k_hs_final<MODE><<<c.red_n, HS_T, smem, s>>>(c, R);
}

int hs_mode(const Ctx& c) {
  // a partitioned plan's pattern table is in global offsets (the march's):
  // its HSCG row sums use the local CSR
  if (!c.pid || c.zm_base) return 0;
  if (c.pid_bytes == 1 && c.ss_ne > 0 && c.hs_ss) return 3;
  return c.pid_bytes == 1 ? 1 : 2;
}
size_t hs_smem(const Ctx& c) {
  if (!c.pid || c.zm_base) return 0;
  return hs_mode(c) == 3 ? ss_smem_bytes(c.pat_np) : pattern_smem_bytes(c.pat_np, c.pat_ne);
}

}  // namespace

void hscg_prepare() {
  const int bytes = 48 * 1024;
#define HS_ATTR(K) cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  HS_ATTR(k_hs_init<1>) HS_ATTR(k_hs_init<2>) HS_ATTR(k_hs_init<3>)
  HS_ATTR((k_hs_ap<1, true>)) HS_ATTR((k_hs_ap<2, true>)) HS_ATTR((k_hs_ap<3, true>))
  HS_ATTR((k_hs_ap<1, false>)) HS_ATTR((k_hs_ap<2, false>)) HS_ATTR((k_hs_ap<3, false>))
  HS_ATTR(k_hs_final<1>) HS_ATTR(k_hs_final<2>) HS_ATTR(k_hs_final<3>)
#undef HS_ATTR
}

void launch_hscg_init(const Ctx& c, double* P, double* R, const double* x0, cudaStream_t s) {
  const size_t smem = hs_smem(c);
  switch (hs_mode(c)) {
    case 3: hs_launch_init<3>(c, P, R, x0, smem, s); break;
    case 1: hs_launch_init<1>(c, P, R, x0, smem, s); break;
    case 2: hs_launch_init<2>(c, P, R, x0, smem, s); break;
    default: hs_launch_init<0>(c, P, R, x0, 0, s); break;
  }
}
void launch_hscg_start(const Ctx& c, cudaStream_t s) { k_hs_start<<<1, 1, 0, s>>>(c); }

// the three kernels of one iteration; the host puts the halo exchange before
// launch_hscg_ap and an allreduce after it and after launch_hscg_xr
void launch_hscg_ap(const Ctx& c, double* P, double* AP, const double* R, bool tv, cudaStream_t s) {
  const size_t smem = hs_smem(c);
  switch (hs_mode(c)) {
    case 3: hs_launch_ap<3>(c, P, AP, R, tv, smem, s); break;
    case 1: hs_launch_ap<1>(c, P, AP, R, tv, smem, s); break;
    case 2: hs_launch_ap<2>(c, P, AP, R, tv, smem, s); break;
    default: hs_launch_ap<0>(c, P, AP, R, tv, 0, s); break;
  }
}
// the two streaming kernels: one wave of 8 CTAs per SM at most, a function of
// the owned rows only (every plan form of an operator sums the same partials)
static int hs_stream_grid(const Ctx& c) {
  const int64_t g = (c.n_own + (int64_t)HS_T * 4 - 1) / ((int64_t)HS_T * 4);
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, RED_BLOCKS));
}
void launch_hscg_xr(const Ctx& c, double* P, double* AP, double* R, bool prod, cudaStream_t s) {
  k_hs_xr<<<hs_stream_grid(c), HS_T, 0, s>>>(c, P, AP, R, prod ? 1 : 0);
}
void launch_hscg_p(const Ctx& c, double* P, double* R, cudaStream_t s) {
  k_hs_p<<<hs_stream_grid(c), HS_T, 0, s>>>(c, P, R);
}
void launch_hscg_final(const Ctx& c, const double* R, cudaStream_t s) {
  const size_t smem = hs_smem(c);
  switch (hs_mode(c)) {
    case 3: hs_launch_final<3>(c, R, smem, s); break;
    case 1: hs_launch_final<1>(c, R, smem, s); break;
    case 2: hs_launch_final<2>(c, R, smem, s); break;
    default: hs_launch_final<0>(c, R, 0, s); break;
  }
}
void launch_hscg_final_row(const Ctx& c, cudaStream_t s) { k_hs_final_row<<<1, 1, 0, s>>>(c); }
