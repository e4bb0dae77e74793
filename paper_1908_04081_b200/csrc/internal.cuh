// internal.cuh -- shared device-side data model of the sm_100a s-step CG path.
//
// Memory layout in HBM (one plan = one operator A on one GPU):
//   CSR       row_ptr int32[n+1], col int32[nnz], val f64[nnz]  (read sigma times/outer)
//   Y         f64 column-major, ld = n rounded up to 32; column l = P_l (l=0..sigma),
//             column sigma+1+l = R_l (l=0..sigma-1).  p and r live IN Y: recovery
//             writes p into column 0 and r into column sigma+1 (row-local, so in place
//             is safe), removing the reference's hstack / Y_t copies (basis.py:239,
//             adaptive.py:166).
//   x, b      f64[n]
//   partials  per-block reduction slots (deterministic fixed-order sums)
//   SolverState  all control state of adaptive_solve (adaptive.py:111-268): the
//             outer loop runs without host round trips; the host only polls `done`.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/sscg.h"

#define SMAX SSCG_MAX_SIGMA   // 16
#define CMAX (2 * SMAX + 1)   // 33 basis columns
#define NB8 ((CMAX + 7) / 8)  // 5 column blocks of 8 (DMMA tiles)
#define GPACK (CMAX * (CMAX + 1) / 2)

// fixed launch geometry (B200: 148 SMs)
#define NUM_SMS 148
#define ROWS_PER_CTA 256
#define RED_BLOCKS (NUM_SMS * 8)   // capacity of the per-CTA partial-sum arrays
#define MT_ROWS 256                 // rows per staged CSR tile (= threads per CTA)
#ifndef MT_STAGES
#define MT_STAGES 2                 // TMA double buffering of CSR tiles
#endif
#define GRAM_BLOCKS (2 * NUM_SMS)  // capacity of the Gram partials
#define SMALL_THREADS 512
#define SS_MAX_NE 8                // union size of the unrolled superset-mask pattern kernels
#define VS_MAX_NE 32               // union size of the value-stream stencil kernels
#ifndef TM_R
#define TM_R 6                     // TMA plane-march ring depth (stages per CTA)
#endif

// TMA tensor maps of the plane march (tmarch.cu): Y as [col][plane][line][x],
// x and b as [plane][line][x], the 1-byte row ids as [plane][line][x]
struct TmMaps {
  CUtensorMap y, x, b, id;
  CUtensorMap y8;  // Y again with a 32 x 8 box (no halo): the two-back vectors of a Chebyshev level
};

struct RitzDev {  // ritz.py:28-158
  double hi_om, hi_h, hi_zeta;
  double lo_om, lo_a, lo_d, lo_g, lo_h;
  double psi, c, eta_next;
  int hi_init, lo_init, count, pad;
};

struct ParamsDev {  // basis.py:39-55
  int kind;
  int has_from;
  double lo, hi;  // generated_from
  double th[SMAX], ga[SMAX], mu[SMAX];
};

struct DevConfig {  // sscg_config + derived constants
  int sigma, s_bar0, f, basis_kind, c_strategy, variant, max_outer, leja_grid;
  int has_bounds, trace_full, n_a, ncols;  // ncols = 2 sigma + 1 (physical Y)
  int solver;       // SSCG_SOLVER_ADAPTIVE / SSCG_SOLVER_FIXED
  int has_fixed;    // fixed solver: caller's parameters below replace params_for
  double fth[SMAX], fga[SMAX], fmu[SMAX];
  double eps_star, bound_lo, bound_hi, norm_a, norm_abs_a, kappa_a;
  int64_t max_iters;  // HSCG: classic.py:47 loop bound
  double unit;      // 2^-53 (ritz.py:25)
  double c0;        // MACHINE_UNIT ** -0.5 (ritz.py:124)
  double nu;        // norm_abs_a / norm_a (adaptive.py:119)
  int64_t cap_iters, cap_outer;
};

struct SolverState {
  int k;          // outer loop index of the block being built
  int done;       // 1: solve finished, every kernel is a no-op
  int status;     // SSCG_RUNNING / CONVERGED / STAGNATED / DIVERGED
  int s_bar;      // degree of the block being built (level kernels read it)
  int s_tilde;
  int s_act;      // inner iterations done in the last block
  int rec_valid;  // recovery applies this outer loop
  int total_iters, total_outer, n_records;
  int best_iter;
  int breakdown;  // non-finite basis column seen (level kernels, atomicOr)
  int first_saved;
  int diag_base;  // global iteration index of the block's first inner iteration
  int gram_count; // last-block-done counter of the Gram kernel
  int diag_n;     // inner iterations of this block needing full-trace diagnostics
  int leja_on;    // Newton parameters of this block still need Leja points 2..sigma-1
  int pad1;
  double best;
  double nb;      // ||b||
  double hs_rr, hs_alpha, hs_beta;  // HSCG scalars (hscg.cu)
  ParamsDev prm;  // parameters of the block being built
  RitzDev rz;
  double cx[CMAX], cr[CMAX], cp[CMAX];      // recovery coefficients, physical columns
  double dx[SMAX][CMAX], dr[SMAX][CMAX];    // per-iteration coords (full trace)
  long long phase_cycles[8];                // K_small phase timers (clock64, thread 0)
};

// everything a kernel may touch; passed by value
struct Ctx {
  const int* rp;
  const int* col;
  const double* val;
  int64_t n;
  int64_t ld;
  double* Y;
  double* x;
  const double* b;
  double* xj;  // full-trace scratch
  double* rj;
  SolverState* st;
  const DevConfig* cfg;
  double* part_t;   // [RED_BLOCKS] ||b - A x||^2 partials
  double* part_r;   // [RED_BLOCKS] ||r||^2 partials
  double* part_d;   // [3][RED_BLOCKS] full-trace partials
  double* part_g;   // [GRAM_BLOCKS][GPACK] Gram partials
  double* leja_obj; // [leja_scratch_doubles] grid objective (two copies) + pairwise-sum state + candidates (small.cu)
  int leja_grid_host;  // cfg->leja_grid as the host knew it at launch / capture
  int leja_split;      // a Leja step as k_leja_grid + k_leja_pick (small operators) or one k_leja_point
  // logs (device)
  double* it_log;   // [cap_iters][SSCG_IT_N]
  int* rec_i;       // [cap_outer][SSCG_REC_NI]
  double* rec_d;    // [cap_outer][SSCG_RECD_ND]
  double* rec_conds;   // [cap_outer][SMAX+1]
  double* rec_th;      // [cap_outer][SMAX]
  double* rec_ga;
  double* rec_mu;
  double* outer_true;  // [cap_outer+1]
  double* first_gram;  // [CMAX*CMAX]
  int red_n;        // CTAs of the row-streaming kernels = partial-sum slots in use
  int stage_cap;    // nnz capacity of one staged CSR tile (0: unstaged kernels)
  // row-slab partition (CA-MPK): local rows are ordered by ghost depth, so the
  // rows a level must (re)compute are a prefix.  Single GPU: every entry == n.
  int64_t n_own;                // owned rows: Gram, recovery, residual norms
  int64_t lvl_rows[SMAX + 1];   // lvl_rows[d] = local rows with ghost depth <= d
  double* red_buf;  // [GPACK + 2] packed Gram + ||b-Ax||^2 + ||r||^2 (allreduced)
  // pattern-compressed operator (plan.cu pattern_setup; NULL pid: CSR kernels).
  // Row i is pattern pid[i]: entries pat_ptr[p] .. pat_ptr[p+1] of
  // (pat_off, pat_val), column = i + pat_off -- A's exact columns, values and
  // stored order, at 1-2 bytes per row instead of 12 per nonzero.
  const void* pid;
  int pid_bytes;     // 1 (<= 256 patterns) or 2
  int pat_np, pat_ne;
  int pat_grid;      // CTAs of the pattern kernels of levels >= 1 (level 0: red_n)
  const int* pat_ptr;
  const int* pat_off;
  const double* pat_val;
  // superset-mask form of the same table (plan.cu superset_setup; ss_ne == 0:
  // not used): every pattern's offsets are a subsequence of the sorted union
  // ss_off[0..ss_ne), so a row is (mask of present union entries, values per
  // union slot).  The offsets travel as kernel parameters (constant bank) and
  // the row loop unrolls fully at compile time.
  // value-stream form (plan.cu vs_setup; vs_ne == 0: not used): a stencil
  // operator whose values vary by row (c4) -- every row's offsets are a
  // subsequence of the sorted union vs_off[0..vs_ne), values stored slot-major
  // vs_val[k * ld + row] (absent slots 0.0): 8 bytes per slot and row, no
  // column indices or row pointers.
  int vs_ne;
  int vs_off[VS_MAX_NE];
  const double* vs_val;
  int vs_sym;  // symmetric form: planes of the diagonal and the upper offsets only (mpk.cu vs_request)
  // a row-partitioned value stream (vs_S > 0): local rows are whole global
  // planes of vs_S rows in a permuted order, so a slot's neighbour is found
  // through plane tables, not by adding the offset: union offset k = vs_dz[k]
  // planes + vs_r[k] rows within the plane; for local block b of vs_S rows,
  // vs_below[b] / vs_above[b] = first local row of the geometric plane below /
  // above it (the block's own first row where that plane is not held -- only
  // absent slots can point there)
  int64_t vs_S;
  int vs_np;
  signed char vs_dz[VS_MAX_NE];
  int vs_r[VS_MAX_NE];
  const int* vs_below;
  const int* vs_above;
  int ss_ne;
  int ss_off[SS_MAX_NE];
  int hs_ss;         // HSCG row sums through the superset mask (SSCG_HS_SS)
  // plane-march form (mpk.cu k_level_zm): the union is symmetric, [-S .. 0 .. S]
  // with S = zm_S >= 256.  Thread t of a CTA owns column c (row mod S) and walks
  // rows c, c + S, c + 2S, ... of one chunk of zm_zc steps, so the -S / 0 / +S
  // entries of a row are the previous step's values (registers) and only one
  // coalesced load per vector per row brings the plane ahead.  zm_S == 0: off.
  int64_t zm_S;
  int zm_zc;       // steps per work item (levels >= 1)
  int zm_zc0;      // steps per work item of level 0 (fixed stripes)
  int64_t zm_items0;
  int zm_ncb;      // column blocks of 256 columns
  int64_t zm_items;  // work items = zm_ncb x ceil(steps / zm_zc)
  int zm_np;         // planes of the walk
  unsigned* zm_ctr;  // [2 (SMAX + 1)] per-level claim / done counters (levels >= 1), or NULL
  const int* zm_base;  // [zm_np] first local row of each plane (partitioned), or NULL (z * S)
  int zm_o;          // 2-D column tiles with line stride zm_o (0: 256 consecutive columns)
  int tm_exact;      // every off-centre pattern value is 0 or +-1: v * x is exact, one fma per term gives the mul + add bits
  // TMA plane march (tmarch.cu; tm == nullptr: the register march): host
  // pointer to the plan's tensor maps (passed to the kernel by value)
  const TmMaps* tm;
  int tm_grid;       // CTAs of its levels >= 1 (level 0: red_n)
  int pf_off;    // pattern kernels: L2 prefetch at row + pf_ahead * stride + pf_off (0: off)
  int pf_ahead;
  const unsigned* ss_mask;  // [pat_np]
  const double* ss_val;     // [pat_np][SS_MAX_NE], absent slots 0
#ifdef SSCG_TIMELINE
  unsigned long long* tl;   // [TL_REPS][TL_NODES][2] first start / last end (globaltimer ns)
#endif
};

// Timeline side build (-DSSCG_TIMELINE, tools/timeline.py): every kernel of the
// outer-loop graph records its first CTA's start and its last warp's end per
// outer loop -- where the time between the kernels goes (there is no nsys here).
#ifdef SSCG_TIMELINE
constexpr int TL_NODES = 40, TL_REPS = 128;
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL_K(c, adj) const int tlk__ = (c).st->k + (adj)
#define TL_BEGIN(c, node)                                                         \
  do {                                                                            \
    if (threadIdx.x == 0 && tlk__ >= 0 && tlk__ < TL_REPS)                        \
      atomicMin(&(c).tl[(tlk__ * TL_NODES + (node)) * 2], tl_now());              \
  } while (0)
#define TL_END(c, node)                                                           \
  do {                                                                            \
    if ((threadIdx.x & 31) == 0 && tlk__ >= 0 && tlk__ < TL_REPS)                 \
      atomicMax(&(c).tl[(tlk__ * TL_NODES + (node)) * 2 + 1], tl_now());          \
  } while (0)
#else
#define TL_K(c, adj)
#define TL_BEGIN(c, node)
#define TL_END(c, node)
#endif

// rows level l must produce for P (ghost depth <= sigma-1-l) and R (<= sigma-2-l)
__host__ __device__ inline int64_t lvl_p_rows(const Ctx& c, int sigma, int l) {
  const int d = sigma - 1 - l;
  return c.lvl_rows[d < 0 ? 0 : d];
}
__host__ __device__ inline int64_t lvl_r_rows(const Ctx& c, int sigma, int l) {
  const int d = sigma - 2 - l;
  return c.lvl_rows[d < 0 ? 0 : d];
}

// the level's column pointers, formed on the host: kept opaque to the
// compiler's index arithmetic, so each gather is one wide add off a base
// register instead of a re-derived column * ld product
struct ZmPtrs {
  const double* xs[3];
  const double* ym[2];
  double* yo[2];
};

inline ZmPtrs zm_ptrs(const Ctx& c, int l, int sigma) {
  ZmPtrs z;
  const int64_t ld = c.ld;
  if (l == 0) {
    z.xs[0] = c.x;
    z.xs[1] = c.Y;
    z.xs[2] = c.Y + (int64_t)(sigma + 1) * ld;
    z.ym[0] = z.ym[1] = nullptr;
    z.yo[0] = c.Y + ld;
    z.yo[1] = c.Y + (int64_t)(sigma + 2) * ld;
  } else {
    z.xs[0] = c.Y + (int64_t)l * ld;
    z.xs[1] = c.Y + (int64_t)(sigma + 1 + l) * ld;
    z.xs[2] = nullptr;
    z.ym[0] = z.xs[0] - ld;
    z.ym[1] = z.xs[1] - ld;
    z.yo[0] = c.Y + (int64_t)(l + 1) * ld;
    z.yo[1] = c.Y + (int64_t)(sigma + 2 + l) * ld;
  }
  return z;
}

// halo exchange lists of a row-partitioned plan (dist.cu)
struct HaloPlan {
  int n_peers = 0;
  int* peer_rank = nullptr;     // host [n_peers]
  int64_t* send_off = nullptr;  // host [n_peers + 1] (rows)
  int64_t* recv_off = nullptr;  // host [n_peers + 1]
  int n_send = 0, n_recv = 0;
  int* d_send_idx = nullptr;    // owned local rows to send, grouped by peer
  int* d_send_dst = nullptr;    // their offset in the send buffer ([p | r | x] per peer)
  int* d_send_cnt = nullptr;    // the peer segment's row count
  int* d_recv_idx = nullptr;    // ghost local rows, grouped by peer
  int* d_recv_src = nullptr;
  int* d_recv_cnt = nullptr;
  double* d_sendbuf = nullptr;  // [3 n_send]
  double* d_recvbuf = nullptr;  // [3 n_recv]
  int r_col = 0;                // physical column of R_0 (sigma + 1) of the current run
};

// Kernel attributes (dynamic shared-memory ceilings) are per device: a
// process that drives several GPUs (adaptive_solve(device=k), the
// single-process multi-GPU group) must set them on each.  Returns true the
// first time it is called for the current device with this mask (the caller
// then sets its attributes); concurrent callers may both see true (setting an
// attribute twice is harmless).
inline bool first_use_on_device(std::atomic<unsigned long long>& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  return (mask.load(std::memory_order_acquire) & bit) == 0;
}
inline void mark_device_done(std::atomic<unsigned long long>& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  mask.fetch_or(1ull << (dev & 63), std::memory_order_release);
}

// Device-side bounds checks of the checked side build (-DSSCG_CHECKED, the
// stand-in for compute-sanitizer, which this pool does not offer): a violated
// index traps with a kernel fault the host reports.  Compiled out otherwise.
#ifdef SSCG_CHECKED
#define SSCG_CHECK(cond)   \
  do {                     \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define SSCG_CHECK(cond) \
  do {                   \
  } while (0)
#endif

#define CUDA_OK(expr)                                             \
  do {                                                            \
    cudaError_t e__ = (expr);                                     \
    if (e__ != cudaSuccess) return sscg_fail_cuda(e__, #expr);    \
  } while (0)

int sscg_fail_cuda(cudaError_t e, const char* what);
int sscg_fail(int code, const char* fmt, ...);

// ---- launchers (defined in the .cu files) ----
// mpk.cu
void launch_init_residual(const Ctx& c, const double* x0, cudaStream_t s);
void launch_level(const Ctx& c, int level, int sigma, cudaStream_t s);
void launch_spmv(const int* rp, const int* col, const double* val, int64_t n, const double* x,
                 double* y, cudaStream_t s);
void launch_block_levels(const int* rp, const int* col, const double* val, int64_t n, int64_t ld,
                         double* Y, int s, const double* th, const double* ga, const double* mu,
                         int* breakdown, cudaStream_t st);
void launch_diag_resid(const Ctx& c, int j, cudaStream_t s);
size_t staged_smem_bytes(int cap);
size_t pattern_smem_bytes(int np, int ne);
void pattern_prepare();
int pattern_ctas_per_sm(int np, int ne, int pid_bytes, int* out2);
size_t ss_smem_bytes(int np);
int ss_ctas_per_sm(int np, int ne, int pid_bytes, int* out2);
int zm_ctas_per_sm(int np, int ne, int pid_bytes, int* out2);
int vs_ctas_per_sm(int ne, bool pl, int* out2);
// tmarch.cu
int tm_make_maps(TmMaps* m, const double* Y, int64_t ld, int ncols, const double* x, const double* b,
                 const void* pid, int64_t o, int64_t S, int64_t planes, int64_t id_planes);
void tm_occupancy(int pat_np, int zm_np, bool table, int* occ0, int* occ1);
void launch_level_tm(const Ctx& c, int level, int sigma, cudaStream_t s);
void staged_prepare(int cap);
int staged_ctas_per_sm(int cap);
// gram.cu (ld must be a multiple of gram_row_multiple(); padding rows zero)
int gram_row_multiple();
void launch_gram(const Ctx& c, int ncols, cudaStream_t s);
void launch_gram_raw(const double* Y, int64_t n, int64_t ld, int k, double* part, double* out,
                     int* counter, cudaStream_t s);
// rec.cu
void launch_recover(const Ctx& c, cudaStream_t s);
void launch_diag_form(const Ctx& c, int j, cudaStream_t s);
void launch_recover_raw(const double* Y, int64_t n, int64_t ld, int k, const double* coef,
                        const double* xbase, double* x, double* r, double* p, cudaStream_t s);
// small.cu
void launch_state_init(const Ctx& c, cudaStream_t s);
void launch_small(const Ctx& c, cudaStream_t s);
void launch_diag_fin(const Ctx& c, int j, cudaStream_t s);
void launch_params_begin(const Ctx& c, cudaStream_t s);
// setup.cu
void launch_pw_apply(const Ctx& c, int mode, double shift, const double* v, double* out,
                     const double* dotv, double* res, cudaStream_t s);
void launch_pw_scale(int64_t n, const double* w, double nw, double* v, cudaStream_t s);
// hscg.cu
void hscg_prepare();
void launch_hscg_init(const Ctx& c, double* P, double* R, const double* x0, cudaStream_t s);
void launch_hscg_start(const Ctx& c, cudaStream_t s);
void launch_hscg_ap(const Ctx& c, double* P, double* AP, const double* R, bool tv, cudaStream_t s);
void launch_hscg_xr(const Ctx& c, double* P, double* AP, double* R, bool prod, cudaStream_t s);
void launch_hscg_p(const Ctx& c, double* P, double* R, cudaStream_t s);
void launch_hscg_final(const Ctx& c, const double* R, cudaStream_t s);
void launch_hscg_final_row(const Ctx& c, cudaStream_t s);
void launch_leja_point(const Ctx& c, int n, cudaStream_t s);
size_t leja_scratch_doubles(int grid);  // Ctx::leja_obj's size (zeroed at allocation)
size_t small_smem_bytes();
// dist.cu
int nccl_load(const char* path);
int nccl_unique_id(const char* path, unsigned char* id128);
int nccl_comm_init(void** comm, const unsigned char* id128, int rank, int world);
void nccl_comm_destroy(void* comm);
int nccl_comm_init_all(void** comms, int n, const int* devs);
void collective_counts(long long* allreduce, long long* halo);
int halo_exchange(const HaloPlan& h, const Ctx& c, void* comm, cudaStream_t s);
void halo_unpack(const HaloPlan& h, const Ctx& c, cudaStream_t s);
int nccl_allreduce(void* comm, double* buf, int64_t count, cudaStream_t s);
void launch_vsum(double* const* d_bufs, int nb, int len, cudaStream_t s);
void launch_norm_pack(const Ctx& c, cudaStream_t s);
int unit_nested_conds(const double* g_host, int s_bar, double* conds_host, int mode, double c,
                      double unit, double eps, double rn, int* s_tilde);
int unit_leja(double lo, double hi, int count, int grid, double* out);
int unit_params_for(int kind, int s, int has, double lo, double hi, int grid, double* th,
                    double* ga, double* mu, int* kind_out);
int unit_ritz(int m, const double* a, const double* b, double* rec);
int unit_sym_eig(int n, const double* m, double* w);
