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
#include "internal.cuh"
#include "ritz.cuh"
#include "rowops.cuh"

namespace {

constexpr int HS_T = ROWS_PER_CTA;  // 256

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

// loop top of classic.py:58-72 for iteration i (thread 0 of the last CTA)
__device__ void hs_classify(SolverState* st, const DevConfig& cf, double true_rel, double r_norm) {
  const int i = st->total_iters;
  int out = SSCG_RUNNING;
  if ((int64_t)i >= cf.max_iters) {
    out = SSCG_EXHAUSTED;  // `while i < max_iters` exits before any verdict
  } else if (true_rel <= cf.eps_star) {
    out = SSCG_CONVERGED;
  } else if (!isfinite(true_rel) || true_rel > 1e5) {
    out = SSCG_DIVERGED;
  } else if (true_rel < st->best) {
    st->best = true_rel;
    st->best_iter = i;
  } else if (i - st->best_iter >= 200 && r_norm <= 0.01 * true_rel * st->nb) {
    out = SSCG_STAGNATED;
  }
  if (out != SSCG_RUNNING) {
    st->status = out;
    st->done = 1;
  }
}

// x = x0, r = b - A x0, p = r; ||b||, r.r; the first loop-top verdict
template <int MODE>
__global__ void __launch_bounds__(HS_T) k_hs_init(Ctx c, double* P, double* R, const double* x0) {
  __shared__ double sm[HS_T / 32];
  RowSum<MODE> A;
  A.init(c);
  SolverState* st = c.st;
  double bb = 0.0, rr = 0.0;
  const int64_t stride = (int64_t)gridDim.x * HS_T;
  for (int64_t i = (int64_t)blockIdx.x * HS_T + threadIdx.x; i < c.n; i += stride) {
    const double bi = c.b[i];
    const double r = __dsub_rn(bi, A.dot(c, i, x0));
    c.x[i] = x0[i];
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
    const DevConfig cf = *c.cfg;
    st->gram_count = 0;
    st->k = 0;
    st->done = 0;
    st->status = SSCG_RUNNING;
    st->total_iters = 0;
    st->total_outer = 0;
    st->n_records = 0;
    st->best = INFINITY;
    st->best_iter = 0;
    st->nb = sqrt(bb);
    st->hs_rr = rr;
    ritz_init(st->rz, cf.c0);
    // the reference's true_vec = b - A x0 is the same computation as r
    hs_classify(st, cf, sqrt(rr) / st->nb, sqrt(rr));
  }
}

template <int MODE>
__global__ void __launch_bounds__(HS_T) k_hs_ap(Ctx c, const double* P, double* AP) {
  __shared__ double sm[HS_T / 32];
  SolverState* st = c.st;
  if (st->done) return;
  RowSum<MODE> A;
  A.init(c);
  double pap = 0.0;
  const int64_t stride = (int64_t)gridDim.x * HS_T;
  for (int64_t i = (int64_t)blockIdx.x * HS_T + threadIdx.x; i < c.n; i += stride) {
    const double ap = A.dot(c, i, P);
    AP[i] = ap;
    pap = fma(P[i], ap, pap);
  }
  pap = block_sum<HS_T>(pap, sm);
  if (threadIdx.x == 0) c.part_t[blockIdx.x] = pap;
  if (!last_cta(&st->gram_count)) return;
  pap = sum_parts(c.part_t, gridDim.x, sm);
  if (threadIdx.x == 0) {
    st->gram_count = 0;
    if (pap <= 0.0 || !isfinite(pap)) {  // classic.py:77-79
      st->status = SSCG_DIVERGED;
      st->done = 1;
    } else {
      st->hs_alpha = st->hs_rr / pap;
    }
  }
}

__global__ void __launch_bounds__(HS_T) k_hs_xr(Ctx c, const double* P, const double* AP,
                                                double* R) {
  __shared__ double sm[HS_T / 32];
  SolverState* st = c.st;
  if (st->done) return;
  const double alpha = st->hs_alpha;
  double rr = 0.0;
  const int64_t stride = (int64_t)gridDim.x * HS_T;
  for (int64_t i = (int64_t)blockIdx.x * HS_T + threadIdx.x; i < c.n; i += stride) {
    c.x[i] = __dadd_rn(c.x[i], __dmul_rn(alpha, P[i]));  // q = alpha*p; x = x + q
    const double r = __dsub_rn(R[i], __dmul_rn(alpha, AP[i]));
    R[i] = r;
    rr = fma(r, r, rr);
  }
  rr = block_sum<HS_T>(rr, sm);
  if (threadIdx.x == 0) c.part_r[blockIdx.x] = rr;
  if (!last_cta(&st->gram_count)) return;
  rr = sum_parts(c.part_r, gridDim.x, sm);
  if (threadIdx.x == 0) {
    st->gram_count = 0;
    const double beta = rr / st->hs_rr;
    const int it = st->total_iters;
    if (double* row = hs_log(c, it)) {
      row[SSCG_IT_ALPHA] = alpha;
      row[SSCG_IT_BETA] = beta;
    }
    ritz_absorb(st->rz, alpha, beta);  // BreakdownSignal -> state untouched
    st->hs_beta = beta;
    st->hs_rr = rr;
    st->total_iters = it + 1;
    st->total_outer = it + 1;  // trace.mark_outer(1) per iteration
  }
}

template <int MODE>
__global__ void __launch_bounds__(HS_T) k_hs_pt(Ctx c, double* P, const double* R) {
  __shared__ double sm[HS_T / 32];
  SolverState* st = c.st;
  if (st->done) return;
  RowSum<MODE> A;
  A.init(c);
  const double beta = st->hs_beta;
  double tt = 0.0, gg = 0.0;
  const int64_t stride = (int64_t)gridDim.x * HS_T;
  for (int64_t i = (int64_t)blockIdx.x * HS_T + threadIdx.x; i < c.n; i += stride) {
    const double r = R[i];
    P[i] = __dadd_rn(r, __dmul_rn(beta, P[i]));
    const double tv = __dsub_rn(c.b[i], A.dot(c, i, c.x));
    const double gv = __dsub_rn(tv, r);
    tt = fma(tv, tv, tt);
    gg = fma(gv, gv, gg);
  }
  tt = block_sum<HS_T>(tt, sm);
  gg = block_sum<HS_T>(gg, sm);
  if (threadIdx.x == 0) {
    c.part_t[blockIdx.x] = tt;
    c.part_d[blockIdx.x] = gg;
  }
  if (!last_cta(&st->gram_count)) return;
  tt = sum_parts(c.part_t, gridDim.x, sm);
  gg = sum_parts(c.part_d, gridDim.x, sm);
  if (threadIdx.x == 0) {
    st->gram_count = 0;
    const DevConfig cf = *c.cfg;
    const double nb = st->nb;
    const double true_rel = sqrt(tt) / nb;
    const double r_norm = sqrt(st->hs_rr);
    if (double* row = hs_log(c, st->total_iters - 1)) {  // trace.record_iteration
      row[SSCG_IT_TRUE] = true_rel;
      row[SSCG_IT_UPD] = r_norm / nb;
      row[SSCG_IT_GAP] = sqrt(gg);
      row[SSCG_IT_XI] = ritz_xi(st->rz);
      row[SSCG_IT_LMIN] = ritz_lmin(st->rz);
      row[SSCG_IT_LMAX] = ritz_lmax(st->rz);
      row[SSCG_IT_PSI] = st->rz.psi;
      row[SSCG_IT_EST] = r_norm / nb;
    }
    hs_classify(st, cf, true_rel, r_norm);
  }
}

template <int MODE>
void hs_launch_init(const Ctx& c, double* P, double* R, const double* x0, size_t smem,
                    cudaStream_t s) {
  k_hs_init<MODE><<<c.red_n, HS_T, smem, s>>>(c, P, R, x0);
}
template <int MODE>
void hs_launch_iter(const Ctx& c, double* P, double* AP, double* R, size_t smem,
                    cudaStream_t s) {
  k_hs_ap<MODE><<<c.red_n, HS_T, smem, s>>>(c, P, AP);
  k_hs_xr<<<c.red_n, HS_T, 0, s>>>(c, P, AP, R);
  k_hs_pt<MODE><<<c.red_n, HS_T, smem, s>>>(c, P, R);
}

int hs_mode(const Ctx& c) {
  if (!c.pid) return 0;
  if (c.pid_bytes == 1 && c.ss_ne > 0 && c.hs_ss) return 3;
  return c.pid_bytes == 1 ? 1 : 2;
}
size_t hs_smem(const Ctx& c) {
  if (!c.pid) return 0;
  return hs_mode(c) == 3 ? ss_smem_bytes(c.pat_np) : pattern_smem_bytes(c.pat_np, c.pat_ne);
}

}  // namespace

void hscg_prepare() {
  const int bytes = 48 * 1024;
  cudaFuncSetAttribute(k_hs_init<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_hs_init<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_hs_ap<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_hs_ap<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_hs_pt<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_hs_pt<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_hs_init<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_hs_ap<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_hs_pt<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
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

void launch_hscg_iter(const Ctx& c, double* P, double* AP, double* R, cudaStream_t s) {
  const size_t smem = hs_smem(c);
  switch (hs_mode(c)) {
    case 3: hs_launch_iter<3>(c, P, AP, R, smem, s); break;
    case 1: hs_launch_iter<1>(c, P, AP, R, smem, s); break;
    case 2: hs_launch_iter<2>(c, P, AP, R, smem, s); break;
    default: hs_launch_iter<0>(c, P, AP, R, 0, s); break;
  }
}
