/*
 * sscg.h -- C ABI of the B200-native adaptive s-step CG hot path
 * (arXiv 1908.04081, improved adaptive s-step CG, Alg. 4).
 *
 * Plain C types only (no torch / no CUDA types), caller-owned HOST buffers,
 * integer status codes + a thread-local last-error string, an opaque plan
 * handle.  A plan is not thread-safe; independent plans may be used from
 * different threads (the reference allows concurrent independent solves,
 * SPEC.md:490-491).
 *
 * The reference has no FFI of its own: its boundary is the Python function
 * `sstepcg.adaptive.adaptive_solve(problem, cfg)` (adaptive.py:111) and the
 * helpers it calls.  Each entry point below names the reference interface it
 * replaces; paper_1908_04081_b200/_lib.py binds them with ctypes and
 * INTEGRATION.md shows the stub a maintainer of the reference would add.
 */
#ifndef SSCG_H
#define SSCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSCG_ABI_VERSION 2
#define SSCG_MAX_SIGMA 16 /* 2*sigma+1 <= 33 basis columns */

/* status codes */
#define SSCG_OK 0
#define SSCG_EINVAL 1  /* bad argument (reference: ValueError)            */
#define SSCG_ECUDA 2   /* CUDA runtime / launch failure                   */
#define SSCG_ENOMEM 3  /* device allocation failed                        */
#define SSCG_EPARAM 4  /* basis.py:31 ParameterError                      */
#define SSCG_ENODEV 5  /* no CUDA device: there is no CPU fallback         */
#define SSCG_EBREAKDOWN 6 /* basis.py:35 BasisBreakdownError (non-finite column) */
#define SSCG_EFORMAT 7 /* matio.py:14 MatrixMarketError (line: sscg_mm_error_line) */

/* solve outcome (trace.converged / stagnated / diverged, trace.py:43-45) */
#define SSCG_RUNNING 0
#define SSCG_CONVERGED 1
#define SSCG_STAGNATED 2
#define SSCG_DIVERGED 3
#define SSCG_EXHAUSTED 4  /* fixed s-step: max_outer ran out with no verdict (sstep.py:168-171) */

/* device log capacity (rows past it are not logged; the solve itself is not cut) */
#define SSCG_LOG_CAP_OUTER (1 << 18)
#define SSCG_LOG_CAP_ITERS (1 << 21)

/* sscg_config.solver */
#define SSCG_SOLVER_ADAPTIVE 0  /* adaptive_solve (adaptive.py:111-268)             */
#define SSCG_SOLVER_FIXED 1     /* sstep_solve, fixed s = sigma (sstep.py:79-174)  */

/* basis kinds (basis.py:166-177) and c strategies (ritz.py:184-203) */
#define SSCG_BASIS_MONOMIAL 0
#define SSCG_BASIS_NEWTON 1
#define SSCG_BASIS_CHEBYSHEV 2
#define SSCG_C_ADAPTIVE 0
#define SSCG_C_UNIT 1
#define SSCG_C_KAPPA 2
#define SSCG_C_FULLBOUND 3

/* per-outer integer record columns (OuterLoopRecord, adaptive.py:74-86) */
#define SSCG_REC_K 0
#define SSCG_REC_SBAR 1
#define SSCG_REC_STILDE 2
#define SSCG_REC_SACTUAL 3
#define SSCG_REC_BREAKJ 4   /* -1 = None */
#define SSCG_REC_MARK 5     /* trace.outer_marks entry */
#define SSCG_REC_PKIND 6    /* basis kind of basis_params_used */
#define SSCG_REC_NI 8
/* per-outer double record columns */
#define SSCG_RECD_PHI 0
#define SSCG_RECD_BLHS 1
#define SSCG_RECD_BRHS 2
#define SSCG_RECD_GEN_LO 3  /* basis_params_used.generated_from (NaN = None) */
#define SSCG_RECD_GEN_HI 4
#define SSCG_RECD_TRUE 5    /* ||b - A x||/||b|| at the start of this outer loop */
#define SSCG_RECD_RREL 6    /* ||r||/||b|| used by select_s_tilde */
#define SSCG_RECD_C 7       /* c_sel used by select_s_tilde */
#define SSCG_RECD_ND 8
/* per-iteration double log columns (SolveTrace.record_iteration, trace.py:50-58) */
#define SSCG_IT_ALPHA 0
#define SSCG_IT_BETA 1
#define SSCG_IT_TRUE 2
#define SSCG_IT_UPD 3
#define SSCG_IT_GAP 4
#define SSCG_IT_XI 5      /* c_values (xi_estimate, ritz.py:154-158) */
#define SSCG_IT_LMIN 6
#define SSCG_IT_LMAX 7
#define SSCG_IT_PSI 8
#define SSCG_IT_EST 9     /* Gram quadrature sqrt(max(0, r'^T G r'))/||b|| */
#define SSCG_IT_N 10

/* AdaptiveConfig (adaptive.py:36-71) + the problem scalars it consults */
typedef struct sscg_config {
  int32_t sigma;
  int32_t s_bar0;
  int32_t f;
  int32_t basis_kind;
  int32_t c_strategy;
  int32_t variant;     /* 0 = old, 1 = improved */
  int32_t max_outer;
  int32_t leja_grid;
  int32_t has_bounds;  /* spectral_bounds given (old variant / monomial path) */
  int32_t trace_full;  /* 1: per-inner-iteration true residual (adaptive.py:205-215) */
  int32_t n_a;         /* max row population (full-bound c) */
  int32_t solver;      /* SSCG_SOLVER_ADAPTIVE / SSCG_SOLVER_FIXED (s = sigma) */
  double eps_star;
  double bound_lo, bound_hi;
  double norm_a, norm_abs_a, kappa_a; /* ProblemInstance scalars (adaptive.py:119,153) */
} sscg_config;

/* Caller-owned host log buffers, filled by sscg_fetch / sscg_solve. */
typedef struct sscg_logs {
  int64_t cap_iters;   /* rows of `iters`                        */
  int64_t cap_outer;   /* rows of rec_i / rec_d / conds / params */
  double* iters;       /* [cap_iters][SSCG_IT_N]                 */
  int32_t* rec_i;      /* [cap_outer][SSCG_REC_NI]                */
  double* rec_d;       /* [cap_outer][SSCG_RECD_ND]               */
  double* conds;       /* [cap_outer][SSCG_MAX_SIGMA+1] cond_used */
  double* thetas;      /* [cap_outer][SSCG_MAX_SIGMA] params used */
  double* gammas;      /* [cap_outer][SSCG_MAX_SIGMA]             */
  double* mus;         /* [cap_outer][SSCG_MAX_SIGMA]             */
  double* outer_true;  /* [cap_outer+1] ||b-Ax||/||b|| at each outer boundary */
  double* first_gram;  /* [(2*sigma+1)^2] first block's G, or NULL */
  /* outputs */
  int32_t status;      /* SSCG_CONVERGED / STAGNATED / DIVERGED / EXHAUSTED */
  int32_t total_iters;
  int32_t total_outer;
  int32_t n_records;   /* len(trace.outer_records)                 */
  int32_t outer_launched; /* outer iterations enqueued (incl. no-op tail) */
  int32_t reserved;
  double device_ms;    /* device time of sscg_run (CUDA events)    */
} sscg_logs;

typedef struct sscg_plan sscg_plan;

const char* sscg_last_error(void);
int sscg_abi_version(void);
int sscg_device_count(int32_t* count);

/* ---- plan: device copy of the CSR operator ---------------------------------
 * Replaces SparseMatrix.as_csr() caching (matio.py:47-53): the matrix is
 * uploaded once per plan and reused by every solve.  row_ptr int64[n+1],
 * col_idx int32[nnz] (sorted per row, as scipy leaves it), values f64[nnz]. */
int sscg_plan_create(sscg_plan** out, int32_t device, int64_t n, int64_t nnz,
                     const int64_t* row_ptr, const int32_t* col_idx, const double* values);
int sscg_plan_destroy(sscg_plan* plan);
/* bytes of device memory the plan holds (matrix + work space) */
int sscg_plan_device_bytes(const sscg_plan* plan, int64_t* bytes);

/* ---- row-partitioned plans (one process per GPU) ----------
 * Local rows are ordered [owned | ghost depth 1 | ... | ghost depth `depth`]
 * (each group in global order), so the rows whose recurrence a matrix-powers
 * level must (redundantly) compute are a prefix: lvl_rows[d] = number of local
 * rows with depth <= d (lvl_rows[0] = n_own, lvl_rows[depth-1] = n_rows,
 * lvl_rows[depth] = n_local).  Rows of depth < depth carry CSR rows (local
 * column indices).  Halo: for peer q (rank peer_rank[q]) the owned local rows
 * send_idx[send_off[q] .. send_off[q+1]) go out and the ghost local rows
 * recv_idx[recv_off[q] .. recv_off[q+1]) come in, both in global row order.
 * Per outer loop: one grouped ncclSend/ncclRecv of p, r, x ghosts and one
 * ncclAllReduce of the packed Gram + residual norms.  nccl_id == NULL builds a
 * member of a single-process virtual group (sscg_vgroup_run) instead. */
typedef struct sscg_part {
  int64_t n_own, n_rows, n_local, nnz;
  int32_t depth;       /* ghost depth provided: solves need sigma <= depth */
  int32_t rank, world;
  int32_t n_peers;
  const int64_t* row_ptr;   /* [n_rows + 1] */
  const int32_t* col_idx;   /* [nnz], local column indices < n_local */
  const double* values;     /* [nnz] */
  const int64_t* lvl_rows;  /* [depth + 1] */
  const int32_t* peer_rank; /* [n_peers] */
  const int64_t* send_off;  /* [n_peers + 1] */
  const int64_t* recv_off;  /* [n_peers + 1] */
  const int32_t* send_idx;  /* [send_off[n_peers]] */
  const int32_t* recv_idx;  /* [recv_off[n_peers]] */
  const unsigned char* nccl_id; /* 128-byte ncclUniqueId shared by the world, or NULL */
  const char* nccl_lib;     /* path of libnccl.so.2 (NULL: default search) */
  const int64_t* global_rows; /* [n_local] global index of each local row, or NULL: lets a
                                 stencil slab keep the plane-march kernels (patterns in
                                 global offsets, planes walked through a table) */
} sscg_part;

int sscg_nccl_unique_id(const char* nccl_lib, unsigned char* id128);
int sscg_plan_create_part(sscg_plan** out, int32_t device, const sscg_part* part);
/* Run a row-partitioned solve of `nplans` plans that all live in this process
 * (on one or more devices) in lock step, exchanging halos with device copies
 * and reducing in fixed order: the multi-rank algorithm without NCCL, for
 * testing it on one GPU.  b[i]: owned rows of plan i; x0[i]: its local rows. */
int sscg_vgroup_run(sscg_plan* const* plans, int32_t nplans, const sscg_config* cfg,
                    const double* const* b, const double* const* x0, sscg_logs* logs0);

/* ---- the solve: adaptive.py:111-268 ---------------------------------------
 * sscg_solve = sscg_load + sscg_run + sscg_fetch (host in, host out). */
int sscg_solve(sscg_plan* plan, const sscg_config* cfg, const double* b, const double* x0,
               double* x_out, sscg_logs* logs);
/* split form: upload b/x0, run entirely on device (inputs resident in HBM;
 * logs->device_ms = CUDA-event time of the run), download x and the logs.
 * Partitioned plans: b and x_out cover the owned rows, x0 every local row. */
int sscg_load(sscg_plan* plan, const double* b, const double* x0);
int sscg_run(sscg_plan* plan, const sscg_config* cfg, sscg_logs* logs);
int sscg_fetch(sscg_plan* plan, double* x_out, sscg_logs* logs);
/* Page-locked host memory for result vectors: an x_out inside such a block is
 * written by one DMA (no staging through bounce buffers).  The Python drop-in
 * keeps a small pool of them behind the arrays adaptive_solve returns (the
 * reference returns a fresh numpy array: adaptive.py:268). */
int sscg_host_alloc(void** out, int64_t bytes);
int sscg_host_free(void* p);
/* per-kernel-class device time of the last sscg_run with profiling enabled:
 * ms[0] mpk level kernels, ms[1] gram, ms[2] small, ms[3] recovery, ms[4] other;
 * counts[] launches of each class.  enable=1 makes the next runs record one
 * event pair per launch (no graph replay). */
int sscg_set_profiling(sscg_plan* plan, int32_t enable);
/* Caller-chosen basis parameters for the fixed s-step solver (sstep_solve's
 * `params`, sstep.py:97-99): theta[s], gamma[s], mu[s-1] (mu may be NULL when
 * s == 1).  They replace params_for(basis_kind, sigma, spectral_bounds) in the
 * next runs with solver == SSCG_SOLVER_FIXED; s must be >= that sigma
 * (ParameterError otherwise, status SSCG_EPARAM).  s == 0 clears them. */
int sscg_set_basis_params(sscg_plan* plan, int32_t s, const double* theta, const double* gamma,
                          const double* mu);
int sscg_get_profile(const sscg_plan* plan, double* ms5, int64_t* counts5);
/* K_small phase timers of the last run (SM clock cycles, thread 0):
 * [0] classify [1] Gram extract + c [2] nested conds [3] s~ + truncation
 * [4] inner loop + record [5] next-block parameters [6] unused [7] calls */
int sscg_get_small_phases(const sscg_plan* plan, int64_t* cycles8);
/* Matrix-powers schedule the plan uses for a given sigma:
 * out[0] 0 = one CSR launch per level, 1 = wavefront passes (SSCG_WAVE=1),
 *        2 = one pattern-compressed launch per level (the default when A's rows
 *        reduce to a small pattern table; SSCG_PATTERN=0 disables);
 * out[1] CTAs; out[2] wavefront dependency reach in row tiles, or the number
 * of row patterns; out[3] passes P; then for q < P: out[4+2q] levels in pass
 * q, out[5+2q] tile lag D of pass q.  out: 4+2*SSCG_MAX_SIGMA int32. */
int sscg_plan_mpk_schedule(sscg_plan* plan, int32_t sigma, int32_t* out);

/* What one outer loop of the plan's captured CUDA graph contains (the graph
 * the last solve built: an s-step outer loop, or one HSCG iteration; -1 before): out[0] ncclAllReduce calls captured into
 * it, out[1] grouped NCCL halo exchanges, out[2] NCCL kernel nodes (by device
 * function name), out[3] kernel nodes, out[4] graph nodes.  A row-partitioned
 * plan must show exactly one allreduce: the algorithm's one synchronisation
 * per outer loop (trace.py:60-64, counted at adaptive.py:178). */
int sscg_plan_collectives(const sscg_plan* plan, int32_t* out5);

/* ---- single-process multi-GPU ------------------------------
 * The drop-in `adaptive_solve(problem, cfg, devices=[...])`: nplans
 * row-partitioned plans in ONE process, plan i (rank i) on devices[i] (distinct
 * GPUs), their NCCL communicators made together by ncclCommInitAll (no
 * unique-id plumbing; parts[i].nccl_id is ignored).  sscg_group_solve runs
 * sscg_solve on every plan concurrently, one host thread and one stream per
 * GPU; b[i] / x_out[i] are rank i's owned rows, x0[i] its local rows, logs[i]
 * its logs (any may be NULL except b).  Destroy each plan with
 * sscg_plan_destroy. */
int sscg_group_create(sscg_plan** plans_out, int32_t nplans, const int32_t* devices,
                      const sscg_part* parts);
int sscg_group_solve(sscg_plan* const* plans, int32_t nplans, const sscg_config* cfg,
                     const double* const* b, const double* const* x0, double* const* x_out,
                     sscg_logs* const* logs);

/* Hestenes-Stiefel CG on the plan's operator (classic.py:33-104 hscg_solve;
 * = sscg_hscg_ex with SSCG_HSCG_REFERENCE).  Every iteration recomputes the true residual b - A x
 * like the reference; logs->iters rows carry alpha, beta, the Ritz values,
 * xi, psi and the true / updated residuals and gap (SSCG_IT_*), at most
 * logs->cap_iters of them; status CONVERGED / STAGNATED / DIVERGED, or
 * EXHAUSTED when max_iters ran out.  max_iters < 0: 100 n. */
int sscg_hscg(sscg_plan* plan, const double* b, const double* x0, double eps_star,
              int64_t max_iters, double* x_out, sscg_logs* logs);
/* HSCG with a choice of semantics, on single-GPU plans and on row-partitioned
 * (NCCL) plans alike -- per iteration one halo exchange of p (and x) and two
 * allreduces (p.Ap with the residual norms; r.r), classic CG's two
 * synchronisations per iteration:
 *   SSCG_HSCG_REFERENCE   classic.py:33-104 (the true residual b - A x every
 *                         iteration drives the verdicts: two SpMVs);
 *   SSCG_HSCG_PRODUCTION  one SpMV per iteration; convergence on the updated
 *                         residual, the true residual formed once at the end
 *                         (the last trace row). */
#define SSCG_HSCG_REFERENCE 0
#define SSCG_HSCG_PRODUCTION 1
int sscg_hscg_ex(sscg_plan* plan, const double* b, const double* x0, double eps_star,
                 int64_t max_iters, int32_t mode, double* x_out, sscg_logs* logs);
/* HSCG over the members of a single-process virtual group (sscg_vgroup_run's
 * plans): lock step, halo by device copies, reductions in fixed order. */
int sscg_vgroup_hscg(sscg_plan* const* plans, int32_t nplans, const double* const* b,
                     const double* const* x0, double eps_star, int64_t max_iters, int32_t mode,
                     sscg_logs* logs0);

/* ---- problem setup (matio.py:104-275) ------------------------------------ */
/* Matrix Market coordinate text -> full symmetric CSR (read_matrix_market,
 * matio.py:104-184): parse `len` bytes (the caller reads / gunzips the file),
 * then copy out row_ptr[n+1], col_idx[nnz], values[nnz] and free.  Errors are
 * SSCG_EFORMAT with the reference's message; sscg_mm_error_line() gives the
 * offending line (0: none). */
typedef struct sscg_mm sscg_mm;
int sscg_mm_parse(const char* text, int64_t len, sscg_mm** mm, int64_t* n, int64_t* nnz,
                  int32_t* symmetric);
int sscg_mm_take(sscg_mm* mm, int64_t* row_ptr, int32_t* col_idx, double* values);
void sscg_mm_free(sscg_mm* mm);
int sscg_mm_error_line(void);
/* _power_iteration (matio.py:229-244) on the device for the plan's operator:
 * mode 0: A v, 1: |A| v, 2: shift * v - A v.  v0 [n] is the normalised start
 * vector (the caller's seeded draw).  Outputs the estimate, the iterations used
 * and whether |lam_k - lam_{k-1}| <= tol |lam_k| was met. */
int sscg_power_iteration(sscg_plan* plan, int32_t mode, double shift, const double* v0,
                         int32_t iters, double tol, double* lam, int32_t* iters_used,
                         int32_t* converged);

/* ---- unit entry points (parity tests; one kernel family each) ------------- */
/* lacore.py:25-34 spmv: y = A x (scipy csr_matvec rounding, bit for bit) */
int sscg_spmv(sscg_plan* plan, const double* x, double* y);
/* basis.py:228-248 build_block without the condition estimates: y_colmajor
 * [(2s+1)][n] (P_0..P_s, R_0..R_{s-1}) and g [(2s+1)^2].  Returns
 * SSCG_EBREAKDOWN on a non-finite column (BasisBreakdownError). */
int sscg_build_block(sscg_plan* plan, const double* p, const double* r, int32_t s,
                     const double* thetas, const double* gammas, const double* mus,
                     double* y_colmajor, double* g);
/* lacore.py:37-47 gram: G = Y^T Y of a column-major n x k block, k <= 33 */
int sscg_gram(int32_t device, int64_t n, int32_t k, const double* y_colmajor, double* g);
/* sstep.py:37-44 recover_iterates: x = x_base + Y xp, r = Y rp, p = Y pp */
int sscg_recover(int32_t device, int64_t n, int32_t k, const double* y_colmajor,
                 const double* xp, const double* rp, const double* pp, const double* x_base,
                 double* x_out, double* r_out, double* p_out);
/* lacore.py:135-148 nested_basis_conds (conds[0] = NaN) */
int sscg_nested_conds(int32_t device, const double* g, int32_t s_bar, double* conds);
/* adaptive.py:89-104 select_s_tilde */
int sscg_select_s_tilde(int32_t device, const double* g, int32_t s_bar, double c, double unit,
                        double eps_star, double r_norm, int32_t* s_tilde, double* conds);
/* basis.py:91-127 leja_points */
int sscg_leja_points(int32_t device, double lmin, double lmax, int32_t count, int32_t grid,
                     double* out);
/* basis.py:166-177 params_for (kind, s, lmin, lmax; has_interval=0 -> None) */
int sscg_params_for(int32_t device, int32_t kind, int32_t s, int32_t has_interval, double lmin,
                    double lmax, int32_t grid, double* thetas, double* gammas, double* mus,
                    int32_t* kind_out);
/* ritz.py:136-158 RitzState.absorb_step over a sequence; rec[m][6] =
 * (lambda_min, lambda_max, psi, c, xi_estimate, count) after each step
 * (nonpositive pairs are skipped, as the callers' BreakdownSignal handlers do) */
int sscg_ritz_sequence(int32_t device, int32_t m, const double* alpha, const double* beta,
                       double* rec);
/* lacore.py:50-100 sym_eig (ascending eigenvalues of a symmetric n x n, n <= 33) */
int sscg_sym_eig(int32_t device, int32_t n, const double* m, double* w);

#ifdef __cplusplus
}
#endif
#endif /* SSCG_H */
