// plan.cu -- host runtime behind the C ABI (include/sscg.h).
//
// A plan owns the device copy of one CSR operator plus every work buffer of the
// solve.  sscg_run drives adaptive_solve (adaptive.py:111-268) entirely on the
// device: one CUDA graph per outer loop (sigma matrix-powers levels, the Gram
// kernel, K_small, [full-trace diagnostics], recovery) is replayed in chunks;
// the host only polls the device `done` word of the previous chunk while the
// next one runs, so the GPU never waits on the host.  Once `done` is set every
// kernel of the remaining replays returns immediately.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "internal.cuh"

void small_prepare();
double sscg_host_c0();

namespace {
thread_local std::string g_err;
constexpr int CHUNK = 4;

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
}  // namespace

int sscg_fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int sscg_fail_cuda(cudaError_t e, const char* what) {
  const int code = (e == cudaErrorMemoryAllocation) ? SSCG_ENOMEM
                   : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) ? SSCG_ENODEV
                                                                                  : SSCG_ECUDA;
  return sscg_fail(code, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

struct sscg_plan {
  int device = 0;
  int64_t n = 0, nnz = 0, ld = 0;
  int* d_rp = nullptr;
  int* d_col = nullptr;
  double* d_val = nullptr;
  int sigma_alloc = 0;
  double* d_Y = nullptr;
  double* d_x = nullptr;
  double* d_b = nullptr;
  double* d_x0 = nullptr;
  double* d_xj = nullptr;
  double* d_rj = nullptr;
  SolverState* d_st = nullptr;
  DevConfig* d_cfg = nullptr;
  double* d_part_t = nullptr;
  double* d_part_r = nullptr;
  double* d_part_d = nullptr;
  double* d_part_g = nullptr;
  double* d_leja = nullptr;
  int leja_cap = 0;
  int64_t cap_iters = 0, cap_outer = 0;
  double* d_it = nullptr;
  int* d_ri = nullptr;
  double* d_rd = nullptr;
  double* d_conds = nullptr;
  double* d_th = nullptr;
  double* d_ga = nullptr;
  double* d_mu = nullptr;
  double* d_otrue = nullptr;
  double* d_fg = nullptr;
  double* d_red = nullptr;  // [GPACK + 2] allreduce payload
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // Leja branch of the outer-loop graph
  cudaEvent_t ev_fork = nullptr;
  int leja_after0 = 1;  // the head chain forks after level 0
  int leja_split = 0;   // small operators: a Leja step over many small CTAs (the chain is their critical path)
  int hs_ss = 1;        // HSCG row sums through the superset mask
  cudaEvent_t ev_leja[SMAX] = {};
  cudaGraphExec_t gexec = nullptr;
  int g_sigma = -1, g_full = -1, g_grid = -1, g_basis = -1;
  // census of the outer-loop graph last built: [0] ncclAllReduce calls, [1]
  // grouped halo exchanges, [2] NCCL kernel nodes, [3] kernel nodes, [4] nodes
  int census[5] = {-1, -1, -1, -1, -1};
  int* h_done = nullptr;  // pinned [2]
  cudaEvent_t ev_chunk[2] = {nullptr, nullptr};
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
  sscg_config cfg{};
  int have_rhs = 0;
  int32_t last_launched = 0;
  double last_ms = 0.0;
  // profiling
  int profiling = 0;
  double prof_ms[5] = {0, 0, 0, 0, 0};
  int64_t prof_cnt[5] = {0, 0, 0, 0, 0};
  int64_t bytes = 0;
  int64_t n_own = 0;               // owned rows (== n on a single-GPU plan)
  int64_t lvl_rows[SMAX + 1] = {};  // local rows with ghost depth <= d
  int red_n = RED_BLOCKS;  // CTAs of the row-streaming kernels
  int stage_cap = 0;       // staged CSR tile capacity (0: unstaged kernels)
  // row partition (sscg_plan_create_part)
  int64_t n_local = 0;     // local rows incl. every ghost depth (vector length)
  int depth = SMAX;        // ghost depth the partition provides (max sigma)
  int rank = 0, world = 1;
  HaloPlan halo;
  void* comm = nullptr;    // ncclComm_t, or NULL (single GPU / virtual group)
  int partitioned = 0;
  // HSCG (sscg_hscg): graph of HS_CHUNK iterations, captured for this Y
  cudaGraphExec_t hs_gexec = nullptr;
  int hs_mode = -1;         // SSCG_HSCG_* the graph was captured for
  double* hs_y = nullptr;   // buffers the captured graph points at
  double* hs_it = nullptr;
  int leja_head = 0;  // Leja chain at the start of the outer loop (small operators)
  // sscg_set_basis_params (fixed s-step solver)
  int fixed_s = 0;
  double fixed_th[SMAX] = {}, fixed_ga[SMAX] = {}, fixed_mu[SMAX] = {};
  // pattern-compressed operator (pattern_setup)
  void* d_pid = nullptr;
  int pid_bytes = 0;
  int pat_np = 0, pat_ne = 0, pat_grid = 0;
  int* d_pat_ptr = nullptr;
  int* d_pat_off = nullptr;
  double* d_pat_val = nullptr;
  int pf_off = 0, pf_ahead = 1;  // L2 prefetch of the pattern kernels (0: off)
  int64_t zm_S = 0;  // plane-march form (0: off)
  int zm_np = 0;
  int* d_zm_base = nullptr;  // plane table of a partitioned march
  unsigned* d_zm_ctr = nullptr;  // dynamic item counters of the level kernels
  int zm_zc = 0, zm_ncb = 0, zm_o = 0, zm_zc0 = 0;
  // TMA plane march (tmarch.cu): on for 2-D-tiled 7-slot marches
  int tm_on = 0, tm_grid = 0;
  int64_t tm_planes = 0, tm_id_planes = 0;
  TmMaps tm{};
  int64_t zm_items0 = 0;
  int64_t zm_items = 0;
  // host <-> device staging of the solve's vectors (copy_h2d / copy_d2h):
  // per copy thread two pinned chunks, a stream and two events
  int st_threads = 0;
  size_t st_chunk = 0;
  std::vector<void*> st_pinned;
  std::vector<cudaStream_t> st_streams;
  std::vector<cudaEvent_t> st_events;
  int vs_ne = 0;  // value-stream stencil form (vs_setup); 0: not used
  int vs_off[VS_MAX_NE] = {};
  double* d_vs_val = nullptr;
  int vs_sym = 0;  // the value stream holds the diagonal's and the upper offsets' planes only
  int64_t vs_S = 0;  // partitioned value stream: plane size (0: plain offsets)
  int vs_np = 0;
  signed char vs_dz[VS_MAX_NE] = {};
  int vs_r[VS_MAX_NE] = {};
  int* d_vs_geo = nullptr;   // vs_below
  int* d_vs_base = nullptr;  // vs_above
  int ss_ne = 0;  // superset-mask form (superset_setup); 0: table-walking kernels
  int ss_exact = 0;  // its off-centre values are all 0 or +-1 (products exact)
  int ss_off[SS_MAX_NE] = {};
  unsigned* d_ss_mask = nullptr;
  double* d_ss_val = nullptr;
};

namespace {

template <class T>
int dalloc(sscg_plan* p, T** ptr, size_t count) {
  if (*ptr) {
    cudaFree(*ptr);
    *ptr = nullptr;
  }
  const size_t b = sizeof(T) * (count ? count : 1);
  CUDA_OK(cudaMalloc((void**)ptr, b));
  p->bytes += (int64_t)b;
  return SSCG_OK;
}

#define TRY(expr)                \
  do {                           \
    int rc__ = (expr);           \
    if (rc__ != SSCG_OK) return rc__; \
  } while (0)

int copy_h2d(sscg_plan* p, void* d, const void* h, size_t bytes);  // staged copies (below)
int copy_d2h(sscg_plan* p, void* h, const void* d, size_t bytes);

int ensure_work(sscg_plan* p, int sigma, int64_t max_outer, int leja_grid) {
  if (sigma > p->sigma_alloc) {
    const int ncols = 2 * sigma + 1;
    TRY(dalloc(p, &p->d_Y, (size_t)p->ld * ncols));
    CUDA_OK(cudaMemset(p->d_Y, 0, sizeof(double) * (size_t)p->ld * ncols));
    p->sigma_alloc = sigma;
    if (p->tm_on)  // the maps point at Y: rebuild them for the new block
      TRY(tm_make_maps(&p->tm, p->d_Y, p->ld, ncols, p->d_x, p->d_b, p->d_pid, p->zm_o, p->zm_S,
                       p->tm_planes, p->tm_id_planes));
    if (p->gexec) {
      cudaGraphExecDestroy(p->gexec);
      p->gexec = nullptr;
    }
  }
  // log capacity is bounded independently of the loop bound (sstep_solve's
  // default max_outer is 100 n / s): rows past it are not logged
  const int64_t co = std::min<int64_t>(max_outer + 2, SSCG_LOG_CAP_OUTER);
  const int64_t ci = std::min<int64_t>((max_outer + 1) * (int64_t)sigma + 1, SSCG_LOG_CAP_ITERS);
  if (co > p->cap_outer || ci > p->cap_iters) {
    const int64_t nco = co > p->cap_outer ? co : p->cap_outer;
    const int64_t nci = ci > p->cap_iters ? ci : p->cap_iters;
    TRY(dalloc(p, &p->d_it, (size_t)nci * SSCG_IT_N));
    TRY(dalloc(p, &p->d_ri, (size_t)nco * SSCG_REC_NI));
    TRY(dalloc(p, &p->d_rd, (size_t)nco * SSCG_RECD_ND));
    TRY(dalloc(p, &p->d_conds, (size_t)nco * (SMAX + 1)));
    TRY(dalloc(p, &p->d_th, (size_t)nco * SMAX));
    TRY(dalloc(p, &p->d_ga, (size_t)nco * SMAX));
    TRY(dalloc(p, &p->d_mu, (size_t)nco * SMAX));
    TRY(dalloc(p, &p->d_otrue, (size_t)nco + 1));
    p->cap_outer = nco;
    p->cap_iters = nci;
    if (p->gexec) {
      cudaGraphExecDestroy(p->gexec);
      p->gexec = nullptr;
    }
  }
  if (leja_grid > p->leja_cap) {
    TRY(dalloc(p, &p->d_leja, leja_scratch_doubles(leja_grid)));  // objective + pairwise-sum state + candidates
    CUDA_OK(cudaMemsetAsync(p->d_leja, 0, 8 * leja_scratch_doubles(leja_grid), p->stream));  // the candidate count
    p->leja_cap = leja_grid;
    if (p->gexec) {
      cudaGraphExecDestroy(p->gexec);
      p->gexec = nullptr;
    }
  }
  return SSCG_OK;
}

#ifdef SSCG_TIMELINE
unsigned long long* g_tl_buf = nullptr;
void tl_reset() {
  const size_t n = (size_t)TL_REPS * TL_NODES;
  std::vector<unsigned long long> h(2 * n);
  for (size_t i = 0; i < n; ++i) {
    h[2 * i] = ~0ull;
    h[2 * i + 1] = 0;
  }
  if (!g_tl_buf) cudaMalloc(&g_tl_buf, sizeof(unsigned long long) * 2 * n);
  cudaMemcpy(g_tl_buf, h.data(), sizeof(unsigned long long) * 2 * n, cudaMemcpyHostToDevice);
}
#endif

Ctx make_ctx(sscg_plan* p) {
  Ctx c;
#ifdef SSCG_TIMELINE
  if (!g_tl_buf) tl_reset();
  c.tl = g_tl_buf;
#endif
  c.rp = p->d_rp;
  c.col = p->d_col;
  c.val = p->d_val;
  c.n = p->n;
  c.ld = p->ld;
  c.Y = p->d_Y;
  c.x = p->d_x;
  c.b = p->d_b;
  c.xj = p->d_xj;
  c.rj = p->d_rj;
  c.st = p->d_st;
  c.cfg = p->d_cfg;
  c.part_t = p->d_part_t;
  c.part_r = p->d_part_r;
  c.part_d = p->d_part_d;
  c.part_g = p->d_part_g;
  c.leja_obj = p->d_leja;
  c.leja_grid_host = p->cfg.leja_grid;
  c.leja_split = p->leja_split;
  c.it_log = p->d_it;
  c.rec_i = p->d_ri;
  c.rec_d = p->d_rd;
  c.rec_conds = p->d_conds;
  c.rec_th = p->d_th;
  c.rec_ga = p->d_ga;
  c.rec_mu = p->d_mu;
  c.outer_true = p->d_otrue;
  c.first_gram = p->d_fg;
  c.red_n = p->red_n;
  c.stage_cap = p->stage_cap;
  c.n_own = p->n_own;
  for (int d = 0; d <= SMAX; ++d) c.lvl_rows[d] = p->lvl_rows[d];
  c.red_buf = p->d_red;
  c.pid = p->d_pid;
  c.pid_bytes = p->pid_bytes;
  c.pat_np = p->pat_np;
  c.pat_ne = p->pat_ne;
  c.pat_grid = p->pat_grid;
  c.pat_ptr = p->d_pat_ptr;
  c.pat_off = p->d_pat_off;
  c.pat_val = p->d_pat_val;
  c.tm = p->tm_on ? &p->tm : nullptr;
  c.tm_grid = p->tm_grid;
  c.pf_off = p->pf_off;
  c.pf_ahead = p->pf_ahead;
  c.zm_S = p->zm_S;
  c.zm_zc = p->zm_zc;
  c.zm_ncb = p->zm_ncb;
  c.zm_items = p->zm_items;
  c.zm_zc0 = p->zm_zc0;
  c.zm_items0 = p->zm_items0;
  c.zm_np = p->zm_np;
  c.zm_base = p->d_zm_base;
  c.zm_ctr = p->d_zm_ctr;
  c.zm_o = p->zm_o;
  c.tm_exact = p->ss_exact;
  c.vs_ne = p->vs_ne;
  for (int k = 0; k < VS_MAX_NE; ++k) c.vs_off[k] = p->vs_off[k];
  c.vs_val = p->d_vs_val;
  c.vs_sym = p->vs_sym;
  c.vs_S = p->vs_S;
  c.vs_np = p->vs_np;
  for (int k = 0; k < VS_MAX_NE; ++k) {
    c.vs_dz[k] = p->vs_dz[k];
    c.vs_r[k] = p->vs_r[k];
  }
  c.vs_below = p->d_vs_geo;
  c.vs_above = p->d_vs_base;
  c.ss_ne = p->ss_ne;
  c.hs_ss = p->hs_ss;
  for (int k = 0; k < SS_MAX_NE; ++k) c.ss_off[k] = p->ss_off[k];
  c.ss_mask = p->d_ss_mask;
  c.ss_val = p->d_ss_val;
  return c;
}

int check_config(const sscg_config* c) {
  if (!c) return sscg_fail(SSCG_EINVAL, "config is NULL");
  if (c->sigma < 1) return sscg_fail(SSCG_EINVAL, "sigma must be >= 1");
  if (c->sigma > SMAX)
    return sscg_fail(SSCG_EINVAL, "sigma=%d exceeds SSCG_MAX_SIGMA=%d", c->sigma, SMAX);
  if (c->s_bar0 < 1 || c->s_bar0 > c->sigma) return sscg_fail(SSCG_EINVAL, "need 1 <= s_bar0 <= sigma");
  if (c->f < 0) return sscg_fail(SSCG_EINVAL, "f must be >= 0");
  if (!(c->eps_star > 0.0)) return sscg_fail(SSCG_EINVAL, "eps_star must be positive");
  if (c->variant != 0 && c->variant != 1) return sscg_fail(SSCG_EINVAL, "unknown variant");
  if (c->basis_kind < 0 || c->basis_kind > 2)
    return sscg_fail(SSCG_EPARAM, "unknown basis kind %d", c->basis_kind);
  if (c->c_strategy < 0 || c->c_strategy > 3)
    return sscg_fail(SSCG_EINVAL, "unknown c strategy %d", c->c_strategy);
  if (c->max_outer < 0) return sscg_fail(SSCG_EINVAL, "max_outer must be >= 0");
  if (c->leja_grid < 2) return sscg_fail(SSCG_EINVAL, "leja_grid must be >= 2");
  if (c->solver != SSCG_SOLVER_ADAPTIVE && c->solver != SSCG_SOLVER_FIXED)
    return sscg_fail(SSCG_EINVAL, "unknown solver %d", c->solver);
  return SSCG_OK;
}

int launch_mpk(sscg_plan* p, const Ctx& c, int sigma, cudaStream_t s);

// Next-block parameters (k_params_begin + Leja points 2..sigma-1) need only the
// Ritz state K_small just updated, so they run on a side branch beside the
// recovery and are joined at the end of the outer loop: the matrix-powers
// kernel of the next outer loop finds every shift ready.  (Outer loop 0 uses
// the initial parameters k_state_init set; params_begin is a no-op there.)
void capture_params_branch(sscg_plan* p, const Ctx& c, int sigma, cudaStream_t s) {
  cudaEventRecord(p->ev_fork, s);
  cudaStreamWaitEvent(p->side, p->ev_fork, 0);
  launch_params_begin(c, p->side);
  for (int n = 2; n < sigma; ++n) launch_leja_point(c, n, p->side);
  cudaEventRecord(p->ev_leja[0], p->side);
}

int capture_outer(sscg_plan* p, const Ctx& c, int sigma, int full, cudaStream_t s) {
  // halo of p, r, x for the communication-avoiding levels (partitioned plans)
  if (p->partitioned && p->comm) {
    TRY(halo_exchange(p->halo, c, p->comm, s));
    halo_unpack(p->halo, c, s);
  }
  if (p->leja_head) {
    // small operators: the recovery is too short to hide the Leja chain, so the
    // chain starts the outer loop on a side branch and level l (l >= 2) joins
    // point l only -- the levels run as the shifts arrive
    launch_params_begin(c, s);
    // the chain forks after level 0 (SSCG_LEJA_AFTER0, default) or before it:
    // level 0 keeps fixed stripes (deterministic norm sums), so a Leja kernel
    // holding one of its SM slots would delay it; level 1 (lambda_min) needs
    // no Leja point, and point 2 (42 us) is ready long before level 2
    const bool after0 = p->leja_after0 && sigma > 1;
    if (after0) launch_level(c, 0, sigma, s);
    // only a Newton basis has a chain (the graph is rebuilt when the basis
    // kind changes); without one the levels follow each other directly
    const bool chain = p->cfg.basis_kind == SSCG_BASIS_NEWTON && sigma > 2;
    if (chain) {
      cudaEventRecord(p->ev_fork, s);
      cudaStreamWaitEvent(p->side, p->ev_fork, 0);
      for (int n = 2; n < sigma; ++n) {
        launch_leja_point(c, n, p->side);
        cudaEventRecord(p->ev_leja[n], p->side);
      }
    }
    for (int l = after0 ? 1 : 0; l < sigma; ++l) {
      if (chain && l >= 2) cudaStreamWaitEvent(s, p->ev_leja[l], 0);
      launch_level(c, l, sigma, s);
    }
  } else {
    TRY(launch_mpk(p, c, sigma, s));
  }
  launch_gram(c, 2 * sigma + 1, s);
  if (p->comm) {  // the one synchronisation of the outer loop
    const int k = 2 * sigma + 1;
    TRY(nccl_allreduce(p->comm, c.red_buf, (int64_t)k * (k + 1) / 2 + 2, s));
  }
  launch_small(c, s);
  const bool tail = !p->leja_head;
  if (tail) capture_params_branch(p, c, sigma, s);
  if (full) {
    for (int j = 0; j < sigma; ++j) {
      launch_diag_form(c, j, s);
      launch_diag_resid(c, j, s);
      launch_diag_fin(c, j, s);
    }
  }
  launch_recover(c, s);
  if (tail) cudaStreamWaitEvent(s, p->ev_leja[0], 0);
  return SSCG_OK;
}

// what the captured outer-loop graph contains: kernel nodes, and among them
// NCCL's (by device-function name) -- the collectives one outer loop issues,
// read back from the graph itself
void graph_census(cudaGraph_t g, int* census) {
  size_t nn = 0;
  census[2] = census[3] = census[4] = 0;
  if (cudaGraphGetNodes(g, nullptr, &nn) != cudaSuccess) return;
  std::vector<cudaGraphNode_t> nodes(nn);
  if (nn && cudaGraphGetNodes(g, nodes.data(), &nn) != cudaSuccess) return;
  census[4] = (int)nn;
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nd, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
    ++census[3];
    cudaKernelNodeParams kp;
    const char* name = nullptr;
    if (cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess && kp.func &&
        cudaFuncGetName(&name, kp.func) == cudaSuccess && name &&
        (strstr(name, "nccl") || strstr(name, "NCCL")))
      ++census[2];
  }
  cudaGetLastError();  // a kernel of another library may not resolve by name
}

int build_graph(sscg_plan* p, const Ctx& c, int sigma, int full) {
  if (p->gexec && p->g_sigma == sigma && p->g_full == full && p->g_grid == c.leja_grid_host &&
      p->g_basis == p->cfg.basis_kind)
    return SSCG_OK;
  if (p->gexec) {
    cudaGraphExecDestroy(p->gexec);
    p->gexec = nullptr;
  }
  cudaGraph_t g = nullptr;
  long long ar0, halo0, ar1, halo1;
  collective_counts(&ar0, &halo0);
  // one graph = CHUNK outer loops (the host looks at `done` once per chunk, and
  // an outer loop past the end is a no-op: K_small stops the solve on the
  // device) -- one graph-launch boundary per CHUNK outer loops
  CUDA_OK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
  int crc = SSCG_OK;
  for (int u = 0; u < CHUNK && crc == SSCG_OK; ++u) crc = capture_outer(p, c, sigma, full, p->stream);
  cudaError_t e = cudaStreamEndCapture(p->stream, &g);
  if (crc != SSCG_OK) {
    if (g) cudaGraphDestroy(g);
    return crc;
  }
  if (e != cudaSuccess) return sscg_fail_cuda(e, "cudaStreamEndCapture");
  collective_counts(&ar1, &halo1);
  p->census[0] = (int)((ar1 - ar0) / CHUNK);  // per outer loop
  p->census[1] = (int)((halo1 - halo0) / CHUNK);
  graph_census(g, p->census);
  for (int k = 2; k < 5; ++k) p->census[k] /= CHUNK;
  e = cudaGraphInstantiate(&p->gexec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return sscg_fail_cuda(e, "cudaGraphInstantiate");
  p->g_sigma = sigma;
  p->g_full = full;
  p->g_grid = c.leja_grid_host;
  p->g_basis = p->cfg.basis_kind;
  return SSCG_OK;
}

// profiling mode: launch one outer loop kernel by kernel with event pairs
struct ProfEv {
  int cls;
  int outer;
  cudaEvent_t a, b;
};

int launch_outer_profiled(sscg_plan* p, const Ctx& c, int sigma, int full, int outer,
                          std::vector<ProfEv>& evs) {
  auto rec = [&](int cls, auto&& fn) -> int {
    ProfEv e{cls, outer, nullptr, nullptr};
    CUDA_OK(cudaEventCreate(&e.a));
    CUDA_OK(cudaEventCreate(&e.b));
    CUDA_OK(cudaEventRecord(e.a, p->stream));
    fn();
    CUDA_OK(cudaEventRecord(e.b, p->stream));
    evs.push_back(e);
    return SSCG_OK;
  };
  if (p->partitioned && p->comm) {
    int hrc = SSCG_OK;
    TRY(rec(4, [&] { hrc = halo_exchange(p->halo, c, p->comm, p->stream); halo_unpack(p->halo, c, p->stream); }));
    TRY(hrc);
  }
  int mrc = SSCG_OK;
  TRY(rec(0, [&] { mrc = launch_mpk(p, c, sigma, p->stream); }));
  TRY(mrc);
  TRY(rec(1, [&] { launch_gram(c, 2 * sigma + 1, p->stream); }));
  if (p->comm) {
    const int k = 2 * sigma + 1;
    int arc = SSCG_OK;
    TRY(rec(4, [&] { arc = nccl_allreduce(p->comm, c.red_buf, (int64_t)k * (k + 1) / 2 + 2, p->stream); }));
    TRY(arc);
  }
  TRY(rec(2, [&] { launch_small(c, p->stream); }));
  TRY(rec(4, [&] { launch_params_begin(c, p->stream); }));
  for (int n = 2; n < sigma; ++n) TRY(rec(4, [&] { launch_leja_point(c, n, p->stream); }));
  if (full) {
    for (int j = 0; j < sigma; ++j) {
      TRY(rec(4, [&] { launch_diag_form(c, j, p->stream); }));
      TRY(rec(4, [&] { launch_diag_resid(c, j, p->stream); }));
      TRY(rec(4, [&] { launch_diag_fin(c, j, p->stream); }));
    }
  }
  TRY(rec(3, [&] { launch_recover(c, p->stream); }));
  return SSCG_OK;
}

}  // namespace

extern "C" {

#ifdef SSCG_TIMELINE
// copy out [TL_REPS][TL_NODES][2] and reset (single device, debugging only)
int sscg_debug_timeline(unsigned long long* out, int* reps, int* nodes) {
  cudaDeviceSynchronize();
  *reps = TL_REPS;
  *nodes = TL_NODES;
  if (!g_tl_buf) tl_reset();
  if (out) {
    cudaMemcpy(out, g_tl_buf, sizeof(unsigned long long) * 2 * TL_REPS * TL_NODES,
               cudaMemcpyDeviceToHost);
    tl_reset();
  }
  return (int)cudaGetLastError();
}
#endif

#ifdef SSCG_TIMELINE
// `reps` back-to-back launches of one HBM-bound kernel on the plan's buffers
// (0: Gram of k columns, 1: recovery from k columns): the kernel's time at
// its own steady-state clocks, to compare with its time inside the graph
int sscg_debug_steady(sscg_plan* p, int which, int k, int reps, float* ms_per_launch) {
  cudaSetDevice(p->device);
  double* coef = nullptr;
  cudaMalloc(&coef, sizeof(double) * 3 * CMAX);
  cudaMemset(coef, 0, sizeof(double) * 3 * CMAX);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaMemsetAsync(&p->d_st->gram_count, 0, sizeof(int), p->stream);
  cudaEventRecord(a, p->stream);
  for (int i = 0; i < reps; ++i) {
    if (which == 0)
      launch_gram_raw(p->d_Y, p->n_own, p->ld, k, p->d_part_g, p->d_red, &p->d_st->gram_count, p->stream);
    else
      launch_recover_raw(p->d_Y, p->n_own, p->ld, k, coef, p->d_x, p->d_x, p->d_Y + (int64_t)(p->cfg.sigma + 1) * p->ld,
                         p->d_Y, p->stream);
  }
  cudaEventRecord(b, p->stream);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *ms_per_launch = ms / reps;
  cudaFree(coef);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return (int)cudaGetLastError();
}
#endif

const char* sscg_last_error(void) { return g_err.c_str(); }
int sscg_abi_version(void) { return SSCG_ABI_VERSION; }

int sscg_device_count(int32_t* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return sscg_fail_cuda(e, "cudaGetDeviceCount");
  }
  *count = n;
  return SSCG_OK;
}

}  // extern "C"

namespace {
// shared constructor: n_rows local rows carry matrix rows, n_own of them are
// owned, n_local rows (>= n_rows) is the vector length; lvl[d] = rows with
// ghost depth <= d (d = 0..depth)
const char* env_or(const char* name, const char* dflt);
int copy_h2d(sscg_plan* p, void* d, const void* h, size_t bytes);
int plan_init(sscg_plan* p, int32_t device, int64_t n_rows, int64_t n_own, int64_t n_local,
              int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx, const double* values,
              const int64_t* lvl, int depth) {
  if (n_rows < 1 || n_own < 1 || n_own > n_rows || n_local < n_rows)
    return sscg_fail(SSCG_EINVAL, "n must be >= 1 (n_own <= n_rows <= n_local)");
  if (nnz < 0 || nnz >= ((int64_t)1 << 31))
    return sscg_fail(SSCG_EINVAL, "nnz=%lld outside the int32 CSR range", (long long)nnz);
  if (n_local >= ((int64_t)1 << 31)) return sscg_fail(SSCG_EINVAL, "n exceeds int32 column indices");
  if (!row_ptr || (nnz && (!col_idx || !values))) return sscg_fail(SSCG_EINVAL, "NULL CSR array");
  if (row_ptr[0] != 0 || row_ptr[n_rows] != nnz)
    return sscg_fail(SSCG_EINVAL, "row_ptr must start at 0 and end at nnz");
  int ndev = 0;
  CUDA_OK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return sscg_fail(SSCG_ENODEV, "device %d not present (%d visible)", device, ndev);
  CUDA_OK(cudaSetDevice(device));
  p->device = device;
  p->n = n_rows;
  p->n_own = n_own;
  p->n_local = n_local;
  p->nnz = nnz;
  p->depth = depth;
  p->ld = round_up(n_local, gram_row_multiple());
  for (int d = 0; d <= SMAX; ++d) p->lvl_rows[d] = lvl[d <= depth ? d : depth];
  int rc = SSCG_OK;
  std::vector<int> rp32(n_rows + 1);
  for (int64_t i = 0; i <= n_rows; ++i) {
    if (i && row_ptr[i] < row_ptr[i - 1]) return sscg_fail(SSCG_EINVAL, "row_ptr must be nondecreasing");
    rp32[i] = (int)row_ptr[i];
  }
  // +4 / +2 elements: the staged kernels round bulk copies up to 16 bytes
  TRY(dalloc(p, &p->d_rp, n_rows + 1 + 8));  // +8: 16-byte bulk copies of a tile's row_ptr
  CUDA_OK(cudaMemset(p->d_rp, 0, sizeof(int) * (n_rows + 1 + 8)));
  TRY(dalloc(p, &p->d_col, nnz + 4));
  TRY(dalloc(p, &p->d_val, nnz + 2));
  // the CSR arrays go up through the staged chunk pipelines (pageable host
  // memory: a plain cudaMemcpy of c5w's 1.4 GB takes ~0.4 s)
  CUDA_OK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  CUDA_OK(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
  // (the pipelines' streams do not order after the cudaMemset calls above,
  // which run on the legacy stream and may still be in flight)
  CUDA_OK(cudaDeviceSynchronize());
  TRY(copy_h2d(p, p->d_rp, rp32.data(), sizeof(int) * (size_t)(n_rows + 1)));
  if (nnz) TRY(copy_h2d(p, p->d_col, col_idx, sizeof(int) * (size_t)nnz));
  if (nnz) TRY(copy_h2d(p, p->d_val, values, sizeof(double) * (size_t)nnz));
  for (double** v : {&p->d_x, &p->d_b, &p->d_x0, &p->d_xj, &p->d_rj}) {
    TRY(dalloc(p, v, p->ld));
    CUDA_OK(cudaMemset(*v, 0, sizeof(double) * p->ld));
  }
  TRY(dalloc(p, &p->d_st, 1));
  TRY(dalloc(p, &p->d_cfg, 1));
  TRY(dalloc(p, &p->d_part_t, RED_BLOCKS));
  TRY(dalloc(p, &p->d_part_r, RED_BLOCKS));
  TRY(dalloc(p, &p->d_part_d, 3 * RED_BLOCKS));
  TRY(dalloc(p, &p->d_part_g, (size_t)GRAM_BLOCKS * GPACK));
  TRY(dalloc(p, &p->d_fg, CMAX * CMAX));
  TRY(dalloc(p, &p->d_red, GPACK + 2));
  CUDA_OK(cudaMemset(p->d_st, 0, sizeof(SolverState)));
  CUDA_OK(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
  for (int i = 0; i < SMAX; ++i) CUDA_OK(cudaEventCreateWithFlags(&p->ev_leja[i], cudaEventDisableTiming));
  CUDA_OK(cudaHostAlloc((void**)&p->h_done, 2 * sizeof(int), cudaHostAllocDefault));
  for (auto* ev : {&p->ev_chunk[0], &p->ev_chunk[1]})
    CUDA_OK(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
  CUDA_OK(cudaEventCreate(&p->ev_start));
  CUDA_OK(cudaEventCreate(&p->ev_stop));
  small_prepare();
  hscg_prepare();
  // launch geometry of the row-streaming kernels: TMA-staged CSR tiles when a
  // tile's segment fits shared memory (every stencil), else the direct kernels
  int sms = NUM_SMS;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int64_t maxt = 0;
  for (int64_t r0 = 0; r0 < n_rows; r0 += MT_ROWS) {
    const int64_t r1 = r0 + MT_ROWS < n_rows ? r0 + MT_ROWS : n_rows;
    maxt = std::max<int64_t>(maxt, row_ptr[r1] - row_ptr[r0]);
  }
  const int64_t cap = (maxt + 4 + 3) / 4 * 4;
  const int64_t ntiles = (n_rows + MT_ROWS - 1) / MT_ROWS;
  // staged CSR tiles only while at least 3 CTAs fit an SM (long rows make the
  // tiles large: 27-point rows give 1 CTA/SM, where the direct kernels win)
  const int staged_max = atoi(env_or("SSCG_STAGE_MAX_KB", "200"));  // A/B: 0 = direct kernels
  int per_sm = 0;
  if (staged_smem_bytes((int)cap) <= (size_t)staged_max * 1024) {
    staged_prepare((int)cap);
    per_sm = staged_ctas_per_sm((int)cap);
  }
  if (per_sm >= std::max(1, atoi(env_or("SSCG_STAGE_MIN_CTAS", "3")))) {
    p->stage_cap = (int)cap;
    p->red_n = (int)std::min<int64_t>({(int64_t)sms * per_sm, (int64_t)RED_BLOCKS, ntiles});
  } else {
    p->stage_cap = 0;
    p->red_n = (int)std::min<int64_t>((int64_t)sms * 4, (n_rows + ROWS_PER_CTA - 1) / ROWS_PER_CTA);
  }
  if (p->red_n < 1) p->red_n = 1;
  // where the next block's Leja chain runs (see capture_outer)
  // the Leja chain at the head of the outer loop, level l joining point l:
  // the full-wave recovery (rec.cu) leaves no SM slot for a chain beside it
  // (c5w: 207.7 ms per solve here vs 224.8 beside the recovery, 215.9 with the
  // former 1.33-wave recovery grid); SSCG_LEJA_HEAD=0 restores the side branch
  p->leja_head = atoi(env_or("SSCG_LEJA_HEAD", "1")) != 0;
  p->hs_ss = atoi(env_or("SSCG_HS_SS", "1")) != 0;
  // (c5w: 197.1 vs 198.6 ms; c1, whose levels are shorter than a Leja point,
  // is faster with the fork before level 0: 9.43 vs 9.58 ms)
  p->leja_after0 = atoi(env_or("SSCG_LEJA_AFTER0", n_rows >= ((int64_t)1 << 20) ? "1" : "0")) != 0;
  // beside the level kernels of a large operator the many-CTA grid pass takes
  // SM slots of the next level's single wave (c5w +3 %); there the chain is
  // hidden behind the levels anyway
  p->leja_split = atoi(env_or("SSCG_LEJA_SPLIT", n_rows >= ((int64_t)1 << 20) ? "0" : "1")) != 0;
  return rc;
}

const char* env_or(const char* name, const char* dflt) {
  const char* v = getenv(name);
  return (v && *v) ? v : dflt;
}

// Lossless pattern compression of the operator for the level kernels: rows
// that are translates of each other -- same length, same column offsets
// relative to the row, same values, same stored order -- share one table
// entry.  Used when the table is small (shared memory, 1-2 byte ids);
// otherwise the CSR kernels run.  SSCG_PATTERN=0 disables it (A/B tests).
constexpr int PAT_MAX_BYTES = 16 * 1024;

// Pattern table of the rows: offset(row, col) is col - row (local indices) or,
// for a row-partitioned plan that passes its rows' global indices, grows[col] -
// grows[row] (the slab's rows are translates in the GLOBAL grid even where the
// local ordering -- owned rows, then ghost planes by depth -- is not).  false
// when the table outgrows shared memory.
// Pattern table of the rows [r0, r1): ids local to this table, in order of
// first appearance.  ids32 receives one id per row (index i - r0).
struct PatTable {
  std::vector<int> ptr{0}, off;
  std::vector<double> val;
  std::unordered_map<uint64_t, std::vector<int>> buckets;
  bool ok = true;
  // id of the pattern (offsets o[0..m), values v[0..m)), added if new; -1: table full
  int find_or_add(const int64_t* o, const double* v, int m) {
    uint64_t h = 1469598103934665603ull ^ (uint64_t)m;
    for (int j = 0; j < m; ++j) {
      uint64_t vb;
      std::memcpy(&vb, &v[j], 8);
      h = (h ^ (uint64_t)o[j]) * 1099511628211ull;
      h = (h ^ vb) * 1099511628211ull;
    }
    auto& cand = buckets[h];
    for (int q : cand) {
      const int pb = ptr[(size_t)q], pe = ptr[(size_t)q + 1];
      if (pe - pb != m) continue;
      bool same = true;
      for (int j = 0; j < m && same; ++j)
        same = off[(size_t)(pb + j)] == o[j] && std::memcmp(&val[(size_t)(pb + j)], &v[j], 8) == 0;
      if (same) return q;
    }
    const int id = (int)ptr.size() - 1;
    const size_t ne = off.size() + (size_t)m;
    if (id >= 65535 || ne * 12 + (ptr.size() + 1) * 4 > (size_t)PAT_MAX_BYTES) return -1;
    for (int j = 0; j < m; ++j) {
      if (o[j] != (int64_t)(int)o[j]) return -1;
      off.push_back((int)o[j]);
      val.push_back(v[j]);
    }
    ptr.push_back((int)off.size());
    cand.push_back(id);
    return id;
  }
};

// Rows that are translates of each other (same offsets, values, stored order)
// share a pattern; ids in order of first appearance.  The scan runs on several
// host threads over contiguous row ranges, each with its own table; the tables
// are merged in range order, which keeps first-appearance order (a 256^3
// operator: 1.7 s of plan creation on one thread).
bool build_patterns(int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                    const double* values, const int64_t* grows, std::vector<int>& ptr,
                    std::vector<int>& off, std::vector<double>& val, std::vector<uint16_t>& ids) {
  ids.assign((size_t)n_rows, 0);
  int T = atoi(env_or("SSCG_SETUP_THREADS", "0"));
  if (T <= 0) T = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
  T = (int)std::max<int64_t>(1, std::min<int64_t>(T, n_rows / 65536));
  std::vector<PatTable> tabs((size_t)T);
  std::vector<std::vector<uint16_t>> lid((size_t)T);
  std::atomic<bool> fail{false};
  auto scan = [&](int t) {
    const int64_t r0 = n_rows * t / T, r1 = n_rows * (t + 1) / T;
    PatTable& tb = tabs[(size_t)t];
    std::vector<uint16_t>& li = lid[(size_t)t];
    li.resize((size_t)(r1 - r0));
    std::vector<int64_t> o;
    for (int64_t i = r0; i < r1; ++i) {
      if ((i & 4095) == 0 && fail.load(std::memory_order_relaxed)) return;
      const int64_t b = row_ptr[i], e = row_ptr[i + 1];
      o.resize((size_t)(e - b));
      for (int64_t j = b; j < e; ++j)
        o[(size_t)(j - b)] = grows ? grows[col_idx[j]] - grows[i] : (int64_t)col_idx[j] - i;
      const int id = tb.find_or_add(o.data(), values + b, (int)(e - b));
      if (id < 0) {
        tb.ok = false;
        fail.store(true, std::memory_order_relaxed);
        return;
      }
      li[(size_t)(i - r0)] = (uint16_t)id;
    }
  };
  {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(scan, t);
    scan(0);
    for (auto& x : th) x.join();
  }
  if (fail.load()) return false;
  // merge in range order
  PatTable g;
  std::vector<std::vector<uint16_t>> remap((size_t)T);
  std::vector<int64_t> o;
  for (int t = 0; t < T; ++t) {
    const PatTable& tb = tabs[(size_t)t];
    const int np = (int)tb.ptr.size() - 1;
    remap[(size_t)t].resize((size_t)np);
    for (int q = 0; q < np; ++q) {
      const int pb = tb.ptr[(size_t)q], m = tb.ptr[(size_t)q + 1] - pb;
      o.assign(tb.off.begin() + pb, tb.off.begin() + pb + m);
      const int id = g.find_or_add(o.data(), tb.val.data() + pb, m);
      if (id < 0) return false;
      remap[(size_t)t][(size_t)q] = (uint16_t)id;
    }
  }
  auto apply = [&](int t) {
    const int64_t r0 = n_rows * t / T, r1 = n_rows * (t + 1) / T;
    for (int64_t i = r0; i < r1; ++i) ids[(size_t)i] = remap[(size_t)t][lid[(size_t)t][(size_t)(i - r0)]];
  };
  {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(apply, t);
    apply(0);
    for (auto& x : th) x.join();
  }
  ptr.swap(g.ptr);
  off.swap(g.off);
  val.swap(g.val);
  return true;
}

// The plane-march union: [-S .. 0 .. S], 3, 5 or 7 offsets, S >= 256.
int64_t march_stride(const std::vector<int>& off) {
  std::vector<int> uni(off.begin(), off.end());
  std::sort(uni.begin(), uni.end());
  uni.erase(std::unique(uni.begin(), uni.end()), uni.end());
  const int ne = (int)uni.size();
  if (ne != 3 && ne != 5 && ne != 7) return 0;
  for (int k = 0; k < ne; ++k)
    if (uni[(size_t)k] != -uni[(size_t)(ne - 1 - k)]) return 0;
  return uni.back() >= 256 ? uni.back() : 0;
}

// Local planes of a partitioned plan: every block of S local rows holds one
// whole global plane in global order, and the planes form one contiguous range.
// Returns the local row of each plane's first row in geometric order, or empty.
std::vector<int> plane_bases(int64_t n_local, const int64_t* grows, int64_t S) {
  std::vector<int> none;
  if (S <= 0 || n_local % S != 0) return none;
  const int64_t np = n_local / S;
  int64_t pmin = INT64_MAX;
  for (int64_t b = 0; b < np; ++b) pmin = std::min(pmin, grows[b * S] / S);
  std::vector<int> base((size_t)np, -1);
  for (int64_t b = 0; b < np; ++b) {
    const int64_t g0 = grows[b * S];
    if (g0 % S != 0) return none;
    for (int64_t k = 1; k < S; ++k)
      if (grows[b * S + k] != g0 + k) return none;
    const int64_t z = g0 / S - pmin;
    if (z < 0 || z >= np || base[(size_t)z] >= 0) return none;
    base[(size_t)z] = (int)(b * S);
  }
  return base;
}

int pattern_setup(sscg_plan* p, int64_t n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                  const double* values, const int64_t* grows = nullptr, int64_t n_local = 0) {
  p->d_pid = nullptr;
  if (atoi(env_or("SSCG_PATTERN", "1")) == 0 || n_rows < 1) return SSCG_OK;
  std::vector<int> ptr, off;
  std::vector<double> val;
  std::vector<uint16_t> ids;
  // partitioned: the global-offset table, when its union marches and the local
  // rows are whole global planes; otherwise the local-offset table
  std::vector<int> bases;
  bool ok = false;
  if (grows && atoi(env_or("SSCG_ZM", "1")) != 0 &&
      build_patterns(n_rows, row_ptr, col_idx, values, grows, ptr, off, val, ids)) {
    const int64_t S = march_stride(off);
    bases = plane_bases(n_local, grows, S);
    ok = !bases.empty();
  }
  if (!ok) {
    bases.clear();
    if (!build_patterns(n_rows, row_ptr, col_idx, values, nullptr, ptr, off, val, ids)) return SSCG_OK;
  }
  const int np = (int)ptr.size() - 1, ne = (int)off.size();
  int occ[2] = {0, 0};
  pattern_prepare();
  p->pid_bytes = np <= 256 ? 1 : 2;
  pattern_ctas_per_sm(np, ne, p->pid_bytes, occ);
  if (occ[0] < 1 || occ[1] < 1) return SSCG_OK;
  if (p->pid_bytes == 1) {
    std::vector<uint8_t> i8(ids.begin(), ids.end());
    uint8_t* d = nullptr;
    const size_t padded = (size_t)round_up(n_rows, 256);  // whole tiles for the window kernels' bulk copies
    TRY(dalloc(p, &d, padded));
    CUDA_OK(cudaMemset(d, 0, padded));
    CUDA_OK(cudaMemcpy(d, i8.data(), (size_t)n_rows, cudaMemcpyHostToDevice));
    p->d_pid = d;
  } else {
    uint16_t* d = nullptr;
    const size_t padded = (size_t)round_up(n_rows, 256);
    TRY(dalloc(p, &d, padded));
    CUDA_OK(cudaMemset(d, 0, 2 * padded));
    CUDA_OK(cudaMemcpy(d, ids.data(), 2 * (size_t)n_rows, cudaMemcpyHostToDevice));
    p->d_pid = d;
  }
  TRY(dalloc(p, &p->d_pat_ptr, ptr.size()));
  TRY(dalloc(p, &p->d_pat_off, off.size()));
  TRY(dalloc(p, &p->d_pat_val, val.size()));
  CUDA_OK(cudaMemcpy(p->d_pat_ptr, ptr.data(), 4 * ptr.size(), cudaMemcpyHostToDevice));
  if (ne) {
    CUDA_OK(cudaMemcpy(p->d_pat_off, off.data(), 4 * off.size(), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(p->d_pat_val, val.data(), 8 * val.size(), cudaMemcpyHostToDevice));
  }
  p->pat_np = np;
  p->pat_ne = ne;
  int sms = NUM_SMS;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  const int64_t tiles = (n_rows + ROWS_PER_CTA - 1) / ROWS_PER_CTA;
  p->red_n = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)sms * occ[0], (int64_t)RED_BLOCKS, tiles}));
  p->pat_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * occ[1], tiles));
  // L2 prefetch distance: the largest positive column offset (first touch)
  p->pf_off = 0;
  p->pf_ahead = std::max(1, atoi(env_or("SSCG_PF_AHEAD", "1")));
  if (atoi(env_or("SSCG_PF", "1")) != 0)
    for (int v : off) p->pf_off = std::max(p->pf_off, v);
  // superset-mask form: every pattern sorted by column, union of offsets small
  p->ss_ne = 0;
  if (atoi(env_or("SSCG_PAT_SS", "1")) != 0) {
    std::vector<int> uni(off.begin(), off.end());
    std::sort(uni.begin(), uni.end());
    uni.erase(std::unique(uni.begin(), uni.end()), uni.end());
    // (a union of 1-2 offsets -- a diagonal or bidiagonal operator, L2-sized in
    // the configs -- runs faster on the table walk: c2 46.6k vs 42.7k iter/s)
    bool ok = (int)uni.size() >= 3 && (int)uni.size() <= SS_MAX_NE;
    for (int q = 0; q < np && ok; ++q)
      for (int k = ptr[q] + 1; k < ptr[q + 1] && ok; ++k) ok = off[k - 1] < off[k];
    int socc[2] = {0, 0};
    if (ok) ss_ctas_per_sm(np, (int)uni.size(), p->pid_bytes, socc);
    if (ok && socc[0] >= 1 && socc[1] >= 1) {
      std::vector<unsigned> mask((size_t)np, 0u);
      std::vector<double> sval((size_t)np * SS_MAX_NE, 0.0);
      for (int q = 0; q < np; ++q)
        for (int k = ptr[q]; k < ptr[q + 1]; ++k) {
          const int slot = (int)(std::lower_bound(uni.begin(), uni.end(), off[k]) - uni.begin());
          mask[(size_t)q] |= 1u << slot;
          sval[(size_t)q * SS_MAX_NE + slot] = val[k];
        }
      TRY(dalloc(p, &p->d_ss_mask, mask.size()));
      TRY(dalloc(p, &p->d_ss_val, sval.size()));
      CUDA_OK(cudaMemcpy(p->d_ss_mask, mask.data(), 4 * mask.size(), cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(p->d_ss_val, sval.data(), 8 * sval.size(), cudaMemcpyHostToDevice));
      p->ss_ne = (int)uni.size();
      // Poisson-like operators: a product with 0 or +-1 is exact, so the march
      // may fuse it into its add (same bits as csr_matvec's mul then add)
      p->ss_exact = atoi(env_or("SSCG_TM_EXACT", "1")) != 0;
      for (int q = 0; q < np && p->ss_exact; ++q)
        for (int k = 0; k < (int)uni.size(); ++k) {
          const double v = sval[(size_t)q * SS_MAX_NE + k];
          if (uni[(size_t)k] != 0 && !(v == 0.0 || v == 1.0 || v == -1.0)) p->ss_exact = 0;
        }
      for (int k = 0; k < SS_MAX_NE; ++k) p->ss_off[k] = k < p->ss_ne ? uni[(size_t)k] : 0;
      p->red_n = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)sms * socc[0], (int64_t)RED_BLOCKS, tiles}));
      p->pat_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * socc[1], tiles));
    }
  }
  // plane-march form: a symmetric union [-S .. 0 .. S] of 3, 5 or 7 offsets
  // with S >= 256 (whole coalesced column blocks) and 32-bit row indices
  p->zm_S = 0;
  if (p->ss_ne > 0 && atoi(env_or("SSCG_ZM", "1")) != 0) {
    const int ne = p->ss_ne;
    const int64_t S = p->ss_off[ne - 1];
    bool ok = (ne == 3 || ne == 5 || ne == 7) && S >= 256 && p->ss_off[ne / 2] == 0 &&
              p->ld + S < ((int64_t)1 << 31) && bases.size() <= 4096;
    for (int k = 0; k < ne && ok; ++k) ok = p->ss_off[k] == -p->ss_off[ne - 1 - k];
    int zocc[2] = {0, 0};
    if (ok) zm_ctas_per_sm(np, ne, p->pid_bytes, zocc);
    if (ok && zocc[0] >= 1 && zocc[1] >= 1) {
      // 7-point-like union [-S, -o, -1, 0, 1, o, S] with o a multiple of 32
      // dividing S: 2-D tiles (32 columns x 8 lines of stride o) per work item
      int64_t o = ne == 7 ? p->ss_off[ne - 2] : 0;
      if (!(o >= 32 && o % 32 == 0 && S % o == 0 && p->ss_off[ne - 3] == 1) ||
          atoi(env_or("SSCG_ZM_2D", "1")) == 0)
        o = 0;
      const int64_t ncb = o ? (o / 32) * ((S / o + 7) / 8) : (S + ROWS_PER_CTA - 1) / ROWS_PER_CTA;
      p->zm_o = (int)o;
      // planes of the walk: the partitioned plan's plane table, else ceil(n / S)
      const int64_t steps = bases.empty() ? (n_rows + S - 1) / S : (int64_t)bases.size();
      const int64_t grid = (int64_t)sms * zocc[1];
      int64_t zc = atoi(env_or("SSCG_ZM_ZC", "0"));
      // planes per item: about 1.7 items per resident CTA, at most 24 (c5w:
      // 24 -- 197.9 ms per solve with per-CTA claiming, 202.7 fixed stripes,
      // 204.5 at 16; c3 128^3: 8 -- 27.6 ms, 28.6 at 6, 31.2 at 12)
      const bool dyn = atoi(env_or("SSCG_ZM_DYN", "1")) != 0;
      if (zc <= 0) zc = std::max<int64_t>(2, std::min<int64_t>(24, ncb * steps * 10 / (grid * 17)));
      p->zm_S = S;
      p->zm_np = (int)steps;
      if (!bases.empty()) {
        TRY(dalloc(p, &p->d_zm_base, bases.size()));
        CUDA_OK(cudaMemcpy(p->d_zm_base, bases.data(), 4 * bases.size(), cudaMemcpyHostToDevice));
      }
      p->zm_zc = (int)zc;
      if (dyn) {
        TRY(dalloc(p, &p->d_zm_ctr, 2 * (SMAX + 1)));
        CUDA_OK(cudaMemset(p->d_zm_ctr, 0, sizeof(unsigned) * 2 * (SMAX + 1)));
      }
      p->zm_ncb = (int)ncb;
      p->zm_items = ncb * ((steps + zc - 1) / zc);
      // level 0 keeps fixed stripes: pick the item size whose whole rounds over
      // its grid cost the fewest planes (+1.5 per item for the two prologue
      // loads) -- c5w: 16 (7 rounds) where 24 would leave a partial 5th round
      {
        const int64_t g0 = std::max<int64_t>(1, std::min<int64_t>({(int64_t)sms * zocc[0], (int64_t)RED_BLOCKS}));
        double best = 1e300;
        int64_t zb = zc;
        for (int64_t z = 2; z <= 32; ++z) {
          const int64_t it = ncb * ((steps + z - 1) / z);
          const double cost = (double)((it + g0 - 1) / g0) * ((double)std::min(z, steps) + 1.5);
          if (cost < best - 1e-9) {
            best = cost;
            zb = z;
          }
        }
        const int64_t z0env = atoi(env_or("SSCG_ZM_ZC0", "0"));
        p->zm_zc0 = (int)(z0env > 0 ? z0env : zb);
        p->zm_items0 = ncb * ((steps + p->zm_zc0 - 1) / p->zm_zc0);
      }
      p->red_n = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)sms * zocc[0], (int64_t)RED_BLOCKS, p->zm_items0}));
      p->pat_grid = (int)std::max<int64_t>(1, std::min<int64_t>(grid, p->zm_items));
      // TMA plane march: the 2-D tiled 7-slot form, 1-byte ids, whole planes
      // (SSCG_TM=0: the register march)
      const int64_t nl = bases.empty() ? n_rows : n_local;
      if (o > 0 && ne == 7 && p->pid_bytes == 1 && nl % S == 0 && n_rows % S == 0 &&
          atoi(env_or("SSCG_TM", "1")) != 0) {
        int t0 = 0, t1 = 0;
        tm_occupancy(np, p->zm_np, !bases.empty(), &t0, &t1);
        if (t0 >= 1 && t1 >= 1) {
          p->tm_on = 1;
          p->tm_planes = nl / S;
          p->tm_id_planes = n_rows / S;
          // planes per item of levels >= 1: the producer streams across item
          // boundaries, so items may be longer (each costs two extra planes
          // of staging) -- about 1.7 per CTA, at most 32 (c5w: 32, 1.255 vs
          // 1.288 ms per outer at 24)
          if (atoi(env_or("SSCG_ZM_ZC", "0")) <= 0) {
            const int64_t g1 = (int64_t)sms * t1;
            p->zm_zc = (int)std::max<int64_t>(2, std::min<int64_t>(32, ncb * steps * 10 / (g1 * 17)));
            p->zm_items = ncb * ((steps + p->zm_zc - 1) / p->zm_zc);
          }
          p->red_n = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)sms * t0, (int64_t)RED_BLOCKS, p->zm_items0}));
          p->tm_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * t1, p->zm_items));
        }
      }
    }
  }
  // a global-offset table is only valid for the march (the other kernels
  // add offsets to local rows): without it, fall back to the CSR kernels
  if (!bases.empty() && p->zm_S == 0) {
    p->d_pid = nullptr;
    p->ss_ne = 0;
    return SSCG_OK;
  }
  return SSCG_OK;
}

// Value-stream stencil form for operators whose rows do not compress to
// patterns: every row's column offsets, in stored order, are a strictly
// increasing subsequence of a union of 3..32 offsets -- a stencil's structure
// with row-varying values (c4).  Values go slot-major [k][ld] (absent 0.0).
// A row-partitioned plan passes its rows' global indices: offsets are then
// global, and the local rows must be whole global planes (plane tables; the
// plane size S is the union offset for which they are, with every offset
// decomposing into dz planes + |r| < S / 2 rows).
int vs_setup(sscg_plan* p, int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
             const double* values, const int64_t* grows = nullptr, int64_t n_local = 0) {
  p->vs_ne = 0;
  p->vs_S = 0;
  // SSCG_PATTERN=0 forces the CSR kernels (A/B reference), SSCG_VS=0 this form only
  if (atoi(env_or("SSCG_VS", "1")) == 0 || atoi(env_or("SSCG_PATTERN", "1")) == 0 || n < 1)
    return SSCG_OK;
  auto ofs = [&](int64_t i, int64_t j) -> int64_t {
    return grows ? grows[col_idx[j]] - grows[i] : (int64_t)col_idx[j] - i;
  };
  // the union of offsets, scanned on several host threads over contiguous row
  // ranges (c4: 189 M nonzeros), each with its own sorted set
  int T = atoi(env_or("SSCG_SETUP_THREADS", "0"));
  if (T <= 0) T = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
  T = (int)std::max<int64_t>(1, std::min<int64_t>(T, n / 65536));
  auto on_ranges = [&](auto&& fn) {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(fn, t);
    fn(0);
    for (auto& x : th) x.join();
  };
  std::vector<std::vector<int64_t>> unis((size_t)T);
  std::atomic<bool> bad{false};
  on_ranges([&](int t) {
    std::vector<int64_t>& u = unis[(size_t)t];
    int64_t last = INT64_MIN;  // most rows repeat the previous offset set: skip the search
    for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) {
      if ((i & 4095) == 0 && bad.load(std::memory_order_relaxed)) return;
      int64_t prev = INT64_MIN;
      for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j) {
        const int64_t o = ofs(i, j);
        if (o <= prev) {  // unsorted row
          bad.store(true, std::memory_order_relaxed);
          return;
        }
        prev = o;
        if (o == last) continue;
        last = o;
        auto it = std::lower_bound(u.begin(), u.end(), o);
        if (it == u.end() || *it != o) {
          if ((int)u.size() >= VS_MAX_NE) {
            bad.store(true, std::memory_order_relaxed);
            return;
          }
          u.insert(it, o);
        }
      }
    }
  });
  if (bad.load()) return SSCG_OK;
  std::vector<int64_t> uni;
  for (const auto& u : unis)
    for (int64_t o : u) {
      auto it = std::lower_bound(uni.begin(), uni.end(), o);
      if (it == uni.end() || *it != o) {
        if ((int)uni.size() >= VS_MAX_NE) return SSCG_OK;
        uni.insert(it, o);
      }
    }
  const int ne = (int)uni.size();
  int occ[2] = {0, 0};
  if (ne < 3 || vs_ctas_per_sm(ne, grows != nullptr, occ) < 1) return SSCG_OK;
  std::vector<int> geo, base;
  if (grows) {  // plane tables of the partitioned form
    int64_t S = 0;
    std::vector<int> bases;
    for (int64_t cand : uni) {
      if (cand <= 0 || cand < S) continue;
      bool dec = true;
      for (int64_t o : uni) {
        const int64_t dz = (o >= 0 ? o + cand / 2 : o - cand / 2) / cand, r = o - dz * cand;
        dec = dec && 2 * std::llabs(r) < cand && std::llabs(dz) <= 1;  // neighbour planes only
      }
      if (!dec) continue;
      std::vector<int> b = plane_bases(n_local, grows, cand);
      if (!b.empty()) {
        S = cand;
        bases.swap(b);
      }
    }
    if (S == 0 || (int64_t)bases.size() * S != n_local) return SSCG_OK;
    p->vs_S = S;
    p->vs_np = (int)bases.size();
    base = bases;
    geo.assign(bases.size(), -1);
    for (size_t z = 0; z < bases.size(); ++z) geo[(size_t)(bases[z] / S)] = (int)z;
    for (int k = 0; k < ne; ++k) {
      const int64_t o = uni[(size_t)k];
      const int64_t dz = (o >= 0 ? o + S / 2 : o - S / 2) / S;
      p->vs_dz[k] = (signed char)dz;
      p->vs_r[k] = (int)(o - dz * S);
    }
  }
  // the kernels unroll over a bucket of slots (9 / 18 / 27 / 32): slots past the
  // union exist and hold 0.0.  Each thread zeroes and fills its own row range.
  const int nb = ne <= 9 ? 9 : ne <= 18 ? 18 : ne <= 27 ? 27 : 32;
  const size_t sv_len = (size_t)nb * (size_t)p->ld;
  std::unique_ptr<double[]> sv(new double[sv_len]);
  on_ranges([&](int t) {
    const int64_t r0 = (int64_t)p->ld * t / T, r1 = (int64_t)p->ld * (t + 1) / T;  // incl. padding rows
    for (int k = 0; k < nb; ++k)
      std::memset(sv.get() + (size_t)k * (size_t)p->ld + (size_t)r0, 0, sizeof(double) * (size_t)(r1 - r0));
    for (int64_t i = std::min<int64_t>(r0, n); i < std::min<int64_t>(r1, n); ++i) {
      int k = 0;
      for (int64_t j = row_ptr[i]; j < row_ptr[i + 1]; ++j) {
        const int64_t o = ofs(i, j);
        while (uni[(size_t)k] != o) ++k;  // rows are sorted subsequences of uni
        sv[(size_t)k * (size_t)p->ld + (size_t)i] = values[j];
      }
    }
  });
  if (grows) {
    // per local block: first local rows of the geometric planes below / above
    const size_t nblk = geo.size();
    std::vector<int> below(nblk), above(nblk);
    for (size_t bk = 0; bk < nblk; ++bk) {
      const int zg = geo[bk], own = (int)(bk * (size_t)p->vs_S);
      below[bk] = zg > 0 ? base[(size_t)zg - 1] : own;
      above[bk] = zg + 1 < (int)base.size() ? base[(size_t)zg + 1] : own;
    }
    TRY(dalloc(p, &p->d_vs_geo, nblk));
    TRY(dalloc(p, &p->d_vs_base, nblk));
    CUDA_OK(cudaMemcpy(p->d_vs_geo, below.data(), 4 * nblk, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(p->d_vs_base, above.data(), 4 * nblk, cudaMemcpyHostToDevice));
  }
  // A bitwise symmetric operator (every A[i][i - o] equals A[i - o][i] bit for
  // bit, the union symmetric, no bucket padding) streams half of its planes:
  // the lower offsets read the upper planes o rows earlier (vs_request)
  p->vs_sym = 0;
  if (!grows && ne == nb && (ne & 1) && atoi(env_or("SSCG_VS_SYM", "1")) != 0) {
    const int mid = ne / 2;
    bool sym = uni[(size_t)mid] == 0;
    for (int k = 0; k < mid && sym; ++k) sym = uni[(size_t)k] == -uni[(size_t)(ne - 1 - k)];
    std::atomic<bool> asym{!sym};
    if (sym)
      on_ranges([&](int t) {
        for (int k = 0; k < mid; ++k) {
          const int64_t o = uni[(size_t)k];  // < 0
          const double* lo_p = sv.get() + (size_t)k * (size_t)p->ld;
          const double* up_p = sv.get() + (size_t)(ne - 1 - k) * (size_t)p->ld;
          for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) {
            const int64_t j = i + o;
            const double want = j >= 0 ? up_p[j] : 0.0;
            if (std::memcmp(&lo_p[i], &want, sizeof(double)) != 0) {
              asym.store(true, std::memory_order_relaxed);
              return;
            }
          }
          if (asym.load(std::memory_order_relaxed)) return;
        }
      });
    p->vs_sym = asym.load() ? 0 : 1;
  }
  if (p->vs_sym) {
    const size_t half = (size_t)(ne - ne / 2) * (size_t)p->ld;
    TRY(dalloc(p, &p->d_vs_val, half));
    TRY(copy_h2d(p, p->d_vs_val, sv.get() + (size_t)(ne / 2) * (size_t)p->ld, 8 * half));
  } else {
    TRY(dalloc(p, &p->d_vs_val, sv_len));
    TRY(copy_h2d(p, p->d_vs_val, sv.get(), 8 * sv_len));
  }
  p->vs_ne = ne;
  for (int k = 0; k < VS_MAX_NE; ++k) p->vs_off[k] = k < ne ? (int)uni[(size_t)k] : 0;  // (plain form)
  int sms = NUM_SMS;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  const int64_t tiles = (n + ROWS_PER_CTA - 1) / ROWS_PER_CTA;
  p->red_n = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)sms * occ[0], (int64_t)RED_BLOCKS, tiles}));
  p->pat_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * occ[1], tiles));
  return SSCG_OK;
}

int launch_mpk(sscg_plan* p, const Ctx& c, int sigma, cudaStream_t s) {
  (void)p;
  for (int l = 0; l < sigma; ++l) launch_level(c, l, sigma, s);
  return SSCG_OK;
}

int create_wrapped(sscg_plan** out, const std::function<int(sscg_plan*)>& init) {
  if (!out) return sscg_fail(SSCG_EINVAL, "out is NULL");
  *out = nullptr;
  sscg_plan* p = new sscg_plan();
  const int rc = init(p);
  if (rc != SSCG_OK) {
    std::string keep = g_err;
    sscg_plan_destroy(p);
    g_err = keep;
    return rc;
  }
  *out = p;
  return SSCG_OK;
}
}  // namespace

extern "C" {

int sscg_plan_create(sscg_plan** out, int32_t device, int64_t n, int64_t nnz,
                     const int64_t* row_ptr, const int32_t* col_idx, const double* values) {
  return create_wrapped(out, [&](sscg_plan* p) {
    if (n < 1) return sscg_fail(SSCG_EINVAL, "n must be >= 1");
    int64_t lvl[SMAX + 1];
    for (int d = 0; d <= SMAX; ++d) lvl[d] = n;
    // SSCG_SETUP_TIMING=1: where plan creation spends its time (stderr)
    const bool timing = atoi(env_or("SSCG_SETUP_TIMING", "0")) != 0;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    TRY(plan_init(p, device, n, n, n, nnz, row_ptr, col_idx, values, lvl, SMAX));
    const auto t1 = now();
    TRY(pattern_setup(p, n, row_ptr, col_idx, values));
    const auto t2 = now();
    int rc = SSCG_OK;
    if (!p->d_pid) rc = vs_setup(p, n, row_ptr, col_idx, values);  // else the pattern kernels replace the CSR staging
    if (timing)
      fprintf(stderr, "[sscg] plan_create n=%lld nnz=%lld: init+upload %.1f ms, patterns %.1f ms, value stream %.1f ms\n",
              (long long)n, (long long)nnz, ms(t0, t1), ms(t1, t2), ms(t2, now()));
    return rc;
  });
}

int sscg_nccl_unique_id(const char* nccl_lib, unsigned char* id128) {
  if (!id128) return sscg_fail(SSCG_EINVAL, "NULL id buffer");
  return nccl_unique_id(nccl_lib, id128);
}

int sscg_plan_create_part(sscg_plan** out, int32_t device, const sscg_part* part) {
  return create_wrapped(out, [&](sscg_plan* p) {
    if (!part) return sscg_fail(SSCG_EINVAL, "NULL partition");
    const sscg_part& q = *part;
    if (q.depth < 1 || q.depth > SMAX) return sscg_fail(SSCG_EINVAL, "ghost depth outside [1, %d]", SMAX);
    if (!q.lvl_rows) return sscg_fail(SSCG_EINVAL, "NULL lvl_rows");
    if (q.lvl_rows[0] != q.n_own || q.lvl_rows[q.depth] != q.n_local ||
        q.lvl_rows[q.depth - 1] != q.n_rows)
      return sscg_fail(SSCG_EINVAL, "lvl_rows inconsistent with n_own / n_rows / n_local");
    int rc = plan_init(p, device, q.n_rows, q.n_own, q.n_local, q.nnz, q.row_ptr, q.col_idx,
                       q.values, q.lvl_rows, q.depth);
    if (rc) return rc;
    TRY(pattern_setup(p, q.n_rows, q.row_ptr, q.col_idx, q.values, q.global_rows, q.n_local));
    // no pattern table (row-varying values): the value stream in global offsets
    if (!p->d_pid && q.global_rows)
      TRY(vs_setup(p, q.n_rows, q.row_ptr, q.col_idx, q.values, q.global_rows, q.n_local));
    p->partitioned = 1;
    p->rank = q.rank;
    p->world = q.world;
    HaloPlan& h = p->halo;
    h.n_peers = q.n_peers;
    h.peer_rank = new int[q.n_peers > 0 ? q.n_peers : 1];
    h.send_off = new int64_t[q.n_peers + 1];
    h.recv_off = new int64_t[q.n_peers + 1];
    h.send_off[0] = h.recv_off[0] = 0;
    for (int i = 0; i < q.n_peers; ++i) {
      h.peer_rank[i] = q.peer_rank[i];
      h.send_off[i + 1] = q.send_off[i + 1];
      h.recv_off[i + 1] = q.recv_off[i + 1];
    }
    h.n_send = (int)h.send_off[q.n_peers];
    h.n_recv = (int)h.recv_off[q.n_peers];
    std::vector<int> sdst(h.n_send), scnt(h.n_send), rsrc(h.n_recv), rcnt(h.n_recv);
    for (int i = 0; i < q.n_peers; ++i) {
      for (int64_t t = h.send_off[i]; t < h.send_off[i + 1]; ++t) {
        sdst[t] = (int)(3 * h.send_off[i] + (t - h.send_off[i]));
        scnt[t] = (int)(h.send_off[i + 1] - h.send_off[i]);
      }
      for (int64_t t = h.recv_off[i]; t < h.recv_off[i + 1]; ++t) {
        rsrc[t] = (int)(3 * h.recv_off[i] + (t - h.recv_off[i]));
        rcnt[t] = (int)(h.recv_off[i + 1] - h.recv_off[i]);
      }
    }
    for (int64_t t = 0; t < h.n_send; ++t)
      if (q.send_idx[t] < 0 || q.send_idx[t] >= q.n_own) return sscg_fail(SSCG_EINVAL, "send index not owned");
    for (int64_t t = 0; t < h.n_recv; ++t)
      if (q.recv_idx[t] < q.n_own || q.recv_idx[t] >= q.n_local) return sscg_fail(SSCG_EINVAL, "recv index not a ghost");
    TRY(dalloc(p, &h.d_send_idx, h.n_send));
    TRY(dalloc(p, &h.d_send_dst, h.n_send));
    TRY(dalloc(p, &h.d_send_cnt, h.n_send));
    TRY(dalloc(p, &h.d_recv_idx, h.n_recv));
    TRY(dalloc(p, &h.d_recv_src, h.n_recv));
    TRY(dalloc(p, &h.d_recv_cnt, h.n_recv));
    TRY(dalloc(p, &h.d_sendbuf, 3 * (size_t)h.n_send));
    TRY(dalloc(p, &h.d_recvbuf, 3 * (size_t)h.n_recv));
    if (h.n_send) {
      CUDA_OK(cudaMemcpy(h.d_send_idx, q.send_idx, sizeof(int) * h.n_send, cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(h.d_send_dst, sdst.data(), sizeof(int) * h.n_send, cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(h.d_send_cnt, scnt.data(), sizeof(int) * h.n_send, cudaMemcpyHostToDevice));
    }
    if (h.n_recv) {
      CUDA_OK(cudaMemcpy(h.d_recv_idx, q.recv_idx, sizeof(int) * h.n_recv, cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(h.d_recv_src, rsrc.data(), sizeof(int) * h.n_recv, cudaMemcpyHostToDevice));
      CUDA_OK(cudaMemcpy(h.d_recv_cnt, rcnt.data(), sizeof(int) * h.n_recv, cudaMemcpyHostToDevice));
    }
    if (q.nccl_id) {  // real multi-process run: one NCCL communicator per plan
      TRY(nccl_load(q.nccl_lib));
      TRY(nccl_comm_init(&p->comm, q.nccl_id, q.rank, q.world));
    }
    return SSCG_OK;
  });
}

int sscg_plan_destroy(sscg_plan* p) {
  if (!p) return SSCG_OK;
  cudaSetDevice(p->device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  if (p->gexec) cudaGraphExecDestroy(p->gexec);
  if (p->hs_gexec) cudaGraphExecDestroy(p->hs_gexec);
  if (p->comm) nccl_comm_destroy(p->comm);
  HaloPlan& h = p->halo;
  for (void* b : {(void*)h.d_send_idx, (void*)h.d_send_dst, (void*)h.d_send_cnt, (void*)h.d_recv_idx,
                  (void*)h.d_recv_src, (void*)h.d_recv_cnt, (void*)h.d_sendbuf, (void*)h.d_recvbuf})
    if (b) cudaFree(b);
  delete[] h.peer_rank;
  delete[] h.send_off;
  delete[] h.recv_off;
  void* bufs[] = {p->d_rp, p->d_col, p->d_val, p->d_Y, p->d_x, p->d_b, p->d_x0, p->d_xj,
                  p->d_rj, p->d_st, p->d_cfg, p->d_part_t, p->d_part_r, p->d_part_d,
                  p->d_part_g, p->d_leja, p->d_it, p->d_ri, p->d_rd, p->d_conds, p->d_th,
                  p->d_ga, p->d_mu, p->d_otrue, p->d_fg, p->d_red,
                  p->d_pid, p->d_pat_ptr, p->d_pat_off, p->d_pat_val, p->d_ss_mask, p->d_ss_val,
                  p->d_zm_base, p->d_vs_val, p->d_zm_ctr, p->d_vs_geo, p->d_vs_base};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (p->h_done) cudaFreeHost(p->h_done);
  for (auto ev : {p->ev_chunk[0], p->ev_chunk[1], p->ev_start, p->ev_stop, p->ev_fork})
    if (ev) cudaEventDestroy(ev);
  for (auto ev : p->ev_leja)
    if (ev) cudaEventDestroy(ev);
  for (void* h : p->st_pinned) cudaFreeHost(h);
  for (auto st : p->st_streams) cudaStreamDestroy(st);
  for (auto ev : p->st_events) cudaEventDestroy(ev);
  if (p->stream) cudaStreamDestroy(p->stream);
  if (p->side) cudaStreamDestroy(p->side);
  delete p;
  return SSCG_OK;
}

int sscg_plan_device_bytes(const sscg_plan* p, int64_t* bytes) {
  if (!p || !bytes) return sscg_fail(SSCG_EINVAL, "NULL argument");
  *bytes = p->bytes;
  return SSCG_OK;
}

int sscg_load(sscg_plan* p, const double* b, const double* x0) {
  if (!p || !b) return sscg_fail(SSCG_EINVAL, "NULL argument");
  CUDA_OK(cudaSetDevice(p->device));
  TRY(copy_h2d(p, p->d_b, b, sizeof(double) * p->n_own));
  if (x0)
    TRY(copy_h2d(p, p->d_x0, x0, sizeof(double) * p->n_local));
  else
    CUDA_OK(cudaMemsetAsync(p->d_x0, 0, sizeof(double) * p->n_local, p->stream));
  p->have_rhs = 1;
  return SSCG_OK;
}

int sscg_set_profiling(sscg_plan* p, int32_t enable) {
  if (!p) return sscg_fail(SSCG_EINVAL, "NULL plan");
  p->profiling = enable ? 1 : 0;
  return SSCG_OK;
}

int sscg_set_basis_params(sscg_plan* p, int32_t s, const double* th, const double* ga,
                          const double* mu) {
  if (!p) return sscg_fail(SSCG_EINVAL, "NULL plan");
  if (s == 0) {
    p->fixed_s = 0;
    return SSCG_OK;
  }
  if (s < 0 || !th || !ga || (s > 1 && !mu)) return sscg_fail(SSCG_EINVAL, "bad basis parameters");
  const int keep = s < SMAX ? s : SMAX;  // degrees beyond SSCG_MAX_SIGMA are never used
  for (int i = 0; i < SMAX; ++i) {
    p->fixed_th[i] = i < keep ? th[i] : NAN;
    p->fixed_ga[i] = i < keep ? ga[i] : NAN;
    p->fixed_mu[i] = i < keep - 1 ? mu[i] : NAN;
  }
  p->fixed_s = s;
  return SSCG_OK;
}

int sscg_get_profile(const sscg_plan* p, double* ms5, int64_t* counts5) {
  if (!p || !ms5 || !counts5) return sscg_fail(SSCG_EINVAL, "NULL argument");
  for (int i = 0; i < 5; ++i) {
    ms5[i] = p->prof_ms[i];
    counts5[i] = p->prof_cnt[i];
  }
  return SSCG_OK;
}

}  // extern "C"

namespace {
// ---- host <-> device copies of the solve's vectors --------------------------
// A pageable cudaMemcpy of a 134 MB vector runs at ~10 GB/s (the driver stages
// it through its own pinned buffer, one chunk at a time).  Here T threads each
// own a slice of the vector and pipeline it through two pinned chunks of their
// own: the host memcpy of one chunk overlaps the DMA of the other, and the T
// slices overlap each other.  Small vectors take the plain path.
constexpr size_t STAGE_MIN = (size_t)16 << 20;

int stage_init(sscg_plan* p) {
  if (p->st_threads) return SSCG_OK;
  int t = atoi(env_or("SSCG_COPY_THREADS", "0"));
  if (t <= 0) {
    const unsigned hc = std::thread::hardware_concurrency();
    t = (int)std::min<unsigned>(8u, std::max(1u, hc / 2));
  }
  p->st_chunk = (size_t)4 << 20;
  for (int i = 0; i < t; ++i) {
    cudaStream_t st;
    CUDA_OK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    p->st_streams.push_back(st);
    for (int k = 0; k < 2; ++k) {
      void* h = nullptr;
      CUDA_OK(cudaHostAlloc(&h, p->st_chunk, cudaHostAllocDefault));
      p->st_pinned.push_back(h);
      cudaEvent_t ev;
      CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      p->st_events.push_back(ev);
    }
  }
  p->st_threads = t;
  return SSCG_OK;
}

// every byte of [p, p + len) zero?  (x0 = 0 is the usual start: a chunk of
// zeros is set on the device instead of crossing the host's memory twice and
// PCIe once; any other chunk leaves at its first nonzero word)
bool all_zero(const char* p, size_t len) {
  size_t i = 0;
  for (; i < len && (reinterpret_cast<uintptr_t>(p + i) & 7); ++i)
    if (p[i]) return false;
  const uint64_t* w = reinterpret_cast<const uint64_t*>(p + i);
  const size_t nw = (len - i) / 8;
  size_t k = 0;
  for (; k + 64 <= nw; k += 64) {
    uint64_t acc = 0;
    for (int j = 0; j < 64; ++j) acc |= w[k + j];
    if (acc) return false;
  }
  for (; k < nw; ++k)
    if (w[k]) return false;
  for (i += nw * 8; i < len; ++i)
    if (p[i]) return false;
  return true;
}

int staged_copy(sscg_plan* p, char* dst, const char* src, size_t bytes, bool h2d) {
  if (bytes < STAGE_MIN || atoi(env_or("SSCG_STAGE_COPY", "1")) == 0) {
    CUDA_OK(cudaStreamSynchronize(p->stream));
    CUDA_OK(cudaMemcpy(dst, src, bytes, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost));
    return SSCG_OK;
  }
  {  // a page-locked host side (sscg_host_alloc) takes one DMA, no staging
    cudaPointerAttributes at;
    const void* host = h2d ? (const void*)src : (const void*)dst;
    if (cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost) {
      CUDA_OK(cudaStreamSynchronize(p->stream));
      CUDA_OK(cudaMemcpy(dst, src, bytes, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost));
      return SSCG_OK;
    }
    cudaGetLastError();  // an unregistered pointer may report an error on older drivers
  }
  TRY(stage_init(p));
  CUDA_OK(cudaStreamSynchronize(p->stream));  // device buffers free / results complete
  const int T = p->st_threads;
  const size_t C = p->st_chunk, per = ((bytes + T - 1) / T + 4095) & ~(size_t)4095;  // T * per >= bytes
  std::vector<cudaError_t> err((size_t)T, cudaSuccess);
  auto work = [&](int t) {
    cudaError_t e = cudaSetDevice(p->device);
    const size_t a = std::min(bytes, (size_t)t * per), b = std::min(bytes, a + per);
    cudaStream_t st = p->st_streams[(size_t)t];
    char* pin[2] = {(char*)p->st_pinned[(size_t)2 * t], (char*)p->st_pinned[(size_t)2 * t + 1]};
    cudaEvent_t ev[2] = {p->st_events[(size_t)2 * t], p->st_events[(size_t)2 * t + 1]};
    int k = 0;
    size_t prev_off = 0, prev_len = 0;
    for (size_t off = a; off < b && e == cudaSuccess; off += C, ++k) {
      const size_t len = std::min(C, b - off);
      const int sl = k & 1;
      if (h2d) {
        if (all_zero(src + off, len)) {
          e = cudaMemsetAsync(dst + off, 0, len, st);
          --k;  // no staging slot used
          continue;
        }
        if (k >= 2) e = cudaEventSynchronize(ev[sl]);  // chunk k-2's DMA left this slot
        if (e != cudaSuccess) break;
        std::memcpy(pin[sl], src + off, len);
        e = cudaMemcpyAsync(dst + off, pin[sl], len, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaEventRecord(ev[sl], st);
      } else {
        e = cudaMemcpyAsync(pin[sl], src + off, len, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaEventRecord(ev[sl], st);
        if (e == cudaSuccess && k >= 1) {  // drain chunk k-1 while chunk k is in flight
          e = cudaEventSynchronize(ev[sl ^ 1]);
          if (e == cudaSuccess) std::memcpy(dst + prev_off, pin[sl ^ 1], prev_len);
        }
        prev_off = off;
        prev_len = len;
      }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess && !h2d && k >= 1) std::memcpy(dst + prev_off, pin[(k - 1) & 1], prev_len);
    err[(size_t)t] = e;
  };
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  for (auto e : err) CUDA_OK(e);
  return SSCG_OK;
}

int copy_h2d(sscg_plan* p, void* d, const void* h, size_t bytes) {
  return staged_copy(p, (char*)d, (const char*)h, bytes, true);
}
int copy_d2h(sscg_plan* p, void* h, const void* d, size_t bytes) {
  return staged_copy(p, (char*)h, (const char*)d, bytes, false);
}

// validate, size the work buffers, upload the device config, scrub the logs
int run_prepare(sscg_plan* p, const sscg_config* cfg) {
  if (!p) return sscg_fail(SSCG_EINVAL, "NULL plan");
  TRY(check_config(cfg));
  if (!p->have_rhs) return sscg_fail(SSCG_EINVAL, "sscg_load must precede sscg_run");
  if (p->partitioned && cfg->sigma > p->depth)
    return sscg_fail(SSCG_EINVAL, "sigma=%d exceeds the partition's ghost depth %d", cfg->sigma, p->depth);
  if (p->partitioned && cfg->trace_full)
    return sscg_fail(SSCG_EINVAL, "trace_full is not supported on a row-partitioned solve");
  CUDA_OK(cudaSetDevice(p->device));
  TRY(ensure_work(p, cfg->sigma, cfg->max_outer, cfg->leja_grid));
  p->cfg = *cfg;
  p->halo.r_col = cfg->sigma + 1;
  DevConfig dc;
  memset(&dc, 0, sizeof(dc));
  dc.sigma = cfg->sigma;
  dc.s_bar0 = cfg->s_bar0;
  dc.f = cfg->f;
  dc.basis_kind = cfg->basis_kind;
  dc.c_strategy = cfg->c_strategy;
  dc.variant = cfg->variant;
  dc.max_outer = cfg->max_outer;
  dc.leja_grid = cfg->leja_grid;
  dc.has_bounds = cfg->has_bounds;
  dc.trace_full = cfg->trace_full;
  dc.n_a = cfg->n_a;
  dc.ncols = 2 * cfg->sigma + 1;
  dc.solver = cfg->solver;
  if (cfg->solver == SSCG_SOLVER_FIXED && p->fixed_s > 0) {
    if (p->fixed_s < cfg->sigma)
      return sscg_fail(SSCG_EPARAM, "params cover degree %d, need %d", p->fixed_s, cfg->sigma);
    dc.has_fixed = 1;
    for (int i = 0; i < SMAX; ++i) {
      dc.fth[i] = i < cfg->sigma ? p->fixed_th[i] : NAN;
      dc.fga[i] = i < cfg->sigma ? p->fixed_ga[i] : NAN;
      dc.fmu[i] = i < cfg->sigma - 1 ? p->fixed_mu[i] : NAN;
    }
  }
  dc.eps_star = cfg->eps_star;
  dc.bound_lo = cfg->bound_lo;
  dc.bound_hi = cfg->bound_hi;
  dc.norm_a = cfg->norm_a;
  dc.norm_abs_a = cfg->norm_abs_a;
  dc.kappa_a = cfg->kappa_a;
  dc.unit = std::ldexp(1.0, -53);
  dc.c0 = sscg_host_c0();
  dc.nu = cfg->norm_a != 0.0 ? cfg->norm_abs_a / cfg->norm_a : 1.0;
  dc.cap_iters = p->cap_iters;
  dc.cap_outer = p->cap_outer - 1;
  CUDA_OK(cudaMemcpyAsync(p->d_cfg, &dc, sizeof(dc), cudaMemcpyHostToDevice, p->stream));
  CUDA_OK(cudaMemsetAsync(p->d_it, 0xff, sizeof(double) * p->cap_iters * SSCG_IT_N, p->stream));
  return SSCG_OK;
}
}  // namespace

extern "C" {

int sscg_run(sscg_plan* p, const sscg_config* cfg, sscg_logs* logs) {
  TRY(run_prepare(p, cfg));
  const Ctx c = make_ctx(p);
  const int sigma = cfg->sigma, full = cfg->trace_full ? 1 : 0;
  if (!p->profiling) TRY(build_graph(p, c, sigma, full));

  CUDA_OK(cudaEventRecord(p->ev_start, p->stream));
  launch_init_residual(c, p->d_x0, p->stream);
  launch_norm_pack(c, p->stream);
  if (p->comm) TRY(nccl_allreduce(p->comm, c.red_buf, 1, p->stream));  // ||b||^2 once per solve
  launch_state_init(c, p->stream);
  CUDA_OK(cudaGetLastError());

  const int64_t total = (int64_t)cfg->max_outer + 1;
  int64_t launched = 0;
  int chunk_id = 0;
  std::vector<ProfEv> evs;
  bool finished = false;
  while (launched < total && !finished) {
    const int64_t m = p->profiling ? std::min<int64_t>(total - launched, CHUNK) : CHUNK;
    if (p->profiling) {
      for (int64_t i = 0; i < m; ++i)
        TRY(launch_outer_profiled(p, c, sigma, full, (int)(launched + i), evs));
    } else {
      CUDA_OK(cudaGraphLaunch(p->gexec, p->stream));  // CHUNK outer loops
    }
    launched += m;
    const int slot = chunk_id & 1;
    CUDA_OK(cudaMemcpyAsync(p->h_done + slot, &p->d_st->done, sizeof(int), cudaMemcpyDeviceToHost,
                            p->stream));
    CUDA_OK(cudaEventRecord(p->ev_chunk[slot], p->stream));
    if (chunk_id >= 1) {
      const int prev = slot ^ 1;
      CUDA_OK(cudaEventSynchronize(p->ev_chunk[prev]));
      if (p->h_done[prev]) finished = true;
    }
    ++chunk_id;
  }
  CUDA_OK(cudaEventRecord(p->ev_stop, p->stream));
  CUDA_OK(cudaStreamSynchronize(p->stream));
  CUDA_OK(cudaGetLastError());
  float ms = 0.f;
  CUDA_OK(cudaEventElapsedTime(&ms, p->ev_start, p->ev_stop));
  p->last_ms = ms;
  p->last_launched = (int32_t)launched;
  if (p->profiling) {
    // only outer loops that did work (0..k; later replays are no-op tails)
    int k_done = 0;
    CUDA_OK(cudaMemcpy(&k_done, &p->d_st->k, sizeof(int), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 5; ++i) {
      p->prof_ms[i] = 0.0;
      p->prof_cnt[i] = 0;
    }
    for (auto& e : evs) {
      float t = 0.f;
      cudaEventElapsedTime(&t, e.a, e.b);
      if (e.outer <= k_done) {
        p->prof_ms[e.cls] += t;
        p->prof_cnt[e.cls] += 1;
      }
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
  }
  if (logs) {
    logs->device_ms = ms;
    logs->outer_launched = (int32_t)launched;
  }
  return SSCG_OK;
}

int sscg_fetch(sscg_plan* p, double* x_out, sscg_logs* logs) {
  if (!p) return sscg_fail(SSCG_EINVAL, "NULL plan");
  CUDA_OK(cudaSetDevice(p->device));
  CUDA_OK(cudaStreamSynchronize(p->stream));
  if (x_out) TRY(copy_d2h(p, x_out, p->d_x, sizeof(double) * p->n_own));
  if (!logs) return SSCG_OK;
  SolverState st;
  CUDA_OK(cudaMemcpy(&st, p->d_st, sizeof(st), cudaMemcpyDeviceToHost));
  logs->status = st.status;
  logs->total_iters = st.total_iters;
  logs->total_outer = st.total_outer;
  logs->n_records = st.n_records;
  logs->outer_launched = p->last_launched;
  logs->device_ms = p->last_ms;
  const int64_t ni = std::min<int64_t>({(int64_t)st.total_iters, logs->cap_iters, p->cap_iters});
  const int64_t no = std::min<int64_t>({(int64_t)st.n_records, logs->cap_outer, p->cap_outer});
  if (logs->iters && ni > 0)
    CUDA_OK(cudaMemcpy(logs->iters, p->d_it, sizeof(double) * ni * SSCG_IT_N, cudaMemcpyDeviceToHost));
  if (no > 0) {
    if (logs->rec_i)
      CUDA_OK(cudaMemcpy(logs->rec_i, p->d_ri, sizeof(int) * no * SSCG_REC_NI, cudaMemcpyDeviceToHost));
    if (logs->rec_d)
      CUDA_OK(cudaMemcpy(logs->rec_d, p->d_rd, sizeof(double) * no * SSCG_RECD_ND, cudaMemcpyDeviceToHost));
    if (logs->conds)
      CUDA_OK(cudaMemcpy(logs->conds, p->d_conds, sizeof(double) * no * (SMAX + 1), cudaMemcpyDeviceToHost));
    if (logs->thetas)
      CUDA_OK(cudaMemcpy(logs->thetas, p->d_th, sizeof(double) * no * SMAX, cudaMemcpyDeviceToHost));
    if (logs->gammas)
      CUDA_OK(cudaMemcpy(logs->gammas, p->d_ga, sizeof(double) * no * SMAX, cudaMemcpyDeviceToHost));
    if (logs->mus)
      CUDA_OK(cudaMemcpy(logs->mus, p->d_mu, sizeof(double) * no * SMAX, cudaMemcpyDeviceToHost));
  }
  const int64_t nt = std::min<int64_t>({(int64_t)st.k + 1, logs->cap_outer + 1, p->cap_outer});
  if (logs->outer_true && nt > 0)
    CUDA_OK(cudaMemcpy(logs->outer_true, p->d_otrue, sizeof(double) * nt, cudaMemcpyDeviceToHost));
  if (logs->first_gram && st.first_saved) {
    const int d = 2 * p->cfg.s_bar0 + 1;
    CUDA_OK(cudaMemcpy(logs->first_gram, p->d_fg, sizeof(double) * d * d, cudaMemcpyDeviceToHost));
  }
  return SSCG_OK;
}

int sscg_host_alloc(void** out, int64_t bytes) {
  if (!out || bytes < 1) return sscg_fail(SSCG_EINVAL, "bad host allocation request");
  *out = nullptr;
  cudaError_t e = cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return sscg_fail(SSCG_ENOMEM, "cudaHostAlloc(%lld bytes): %s", (long long)bytes, cudaGetErrorString(e));
  }
  return SSCG_OK;
}
int sscg_host_free(void* p) {
  if (p) cudaFreeHost(p);
  cudaGetLastError();
  return SSCG_OK;
}

int sscg_solve(sscg_plan* p, const sscg_config* cfg, const double* b, const double* x0,
               double* x_out, sscg_logs* logs) {
  TRY(sscg_load(p, b, x0));
  TRY(sscg_run(p, cfg, logs));
  return sscg_fetch(p, x_out, logs);
}

int sscg_get_small_phases(const sscg_plan* p, int64_t* cycles8) {
  if (!p || !cycles8) return sscg_fail(SSCG_EINVAL, "NULL argument");
  CUDA_OK(cudaSetDevice(p->device));
  long long h[8];
  CUDA_OK(cudaMemcpy(h, p->d_st->phase_cycles, sizeof(h), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 8; ++i) cycles8[i] = h[i];
  return SSCG_OK;
}

int sscg_plan_mpk_schedule(sscg_plan* p, int32_t sigma, int32_t* out) {
  if (!p || !out || sigma < 1 || sigma > SMAX) return sscg_fail(SSCG_EINVAL, "bad arguments");
  for (int i = 0; i < 4 + 2 * SMAX; ++i) out[i] = 0;
  out[0] = p->d_pid ? 2 : p->vs_ne ? 3 : 0;
  out[1] = p->red_n;
  out[2] = p->d_pid ? p->pat_np : p->vs_ne;
  // last slot: pattern kernel form (0 table walk, 1 superset mask, 2 plane
  // march, 3 the TMA plane march)
  if (p->d_pid) out[3 + 2 * SMAX] = p->zm_S > 0 ? (p->tm_on ? 3 : 2) : p->ss_ne > 0 ? 1 : 0;
  if (!p->d_pid && p->vs_ne) out[3 + 2 * SMAX] = p->vs_sym;  // value stream: 1 = symmetric form (half the planes)
  if (p->tm_on) out[1] = p->tm_grid;
  out[3] = sigma;
  for (int q = 0; q < sigma; ++q) out[4 + 2 * q] = 1;
  return SSCG_OK;
}

int sscg_plan_collectives(const sscg_plan* p, int32_t* out5) {
  if (!p || !out5) return sscg_fail(SSCG_EINVAL, "NULL argument");
  for (int i = 0; i < 5; ++i) out5[i] = p->census[i];
  return SSCG_OK;
}

// ---- single-process multi-GPU group (one host thread and one
// stream per GPU, communicators from ncclCommInitAll) -------------------------
int sscg_group_create(sscg_plan** out, int32_t nplans, const int32_t* devices,
                      const sscg_part* parts) {
  if (!out || nplans < 1 || !devices || !parts) return sscg_fail(SSCG_EINVAL, "bad group arguments");
  for (int i = 0; i < nplans; ++i) out[i] = nullptr;
  for (int i = 0; i < nplans; ++i)
    for (int j = 0; j < i; ++j)
      if (devices[i] == devices[j])
        return sscg_fail(SSCG_EINVAL, "group devices must be distinct (device %d twice)", devices[i]);
  auto undo = [&](int rc) {
    std::string keep = g_err;
    for (int i = 0; i < nplans; ++i)
      if (out[i]) sscg_plan_destroy(out[i]), out[i] = nullptr;
    g_err = keep;
    return rc;
  };
  for (int i = 0; i < nplans; ++i) {
    if (parts[i].rank != i || parts[i].world != nplans)
      return undo(sscg_fail(SSCG_EINVAL, "part %d is not rank %d of %d", i, i, nplans));
    sscg_part q = parts[i];
    q.nccl_id = nullptr;  // no per-rank init: the group's communicators come below
    const int rc = sscg_plan_create_part(&out[i], devices[i], &q);
    if (rc) return undo(rc);
  }
  int rc = nccl_load(parts[0].nccl_lib);
  if (rc) return undo(rc);
  std::vector<void*> comms((size_t)nplans, nullptr);
  std::vector<int> devs(devices, devices + nplans);
  rc = nccl_comm_init_all(comms.data(), nplans, devs.data());
  if (rc) return undo(rc);
  for (int i = 0; i < nplans; ++i) out[i]->comm = comms[(size_t)i];
  return SSCG_OK;
}

int sscg_group_solve(sscg_plan* const* plans, int32_t nplans, const sscg_config* cfg,
                     const double* const* b, const double* const* x0, double* const* x_out,
                     sscg_logs* const* logs) {
  if (!plans || nplans < 1 || !b) return sscg_fail(SSCG_EINVAL, "bad group arguments");
  for (int i = 0; i < nplans; ++i)
    if (!plans[i] || !plans[i]->comm || plans[i]->rank != i || plans[i]->world != nplans)
      return sscg_fail(SSCG_EINVAL, "plan %d is not rank %d of a %d-GPU group", i, i, nplans);
  // every rank must run concurrently (each outer loop allreduces across all of
  // them): one host thread per GPU, each driving its own plan's stream
  std::vector<int> rcs((size_t)nplans, SSCG_OK);
  std::vector<std::string> errs((size_t)nplans);
  auto run = [&](int i) {
    rcs[(size_t)i] = sscg_solve(plans[i], cfg, b[i], x0 ? x0[i] : nullptr,
                                x_out ? x_out[i] : nullptr, logs ? logs[i] : nullptr);
    if (rcs[(size_t)i]) errs[(size_t)i] = g_err;
  };
  std::vector<std::thread> th;
  for (int i = 1; i < nplans; ++i) th.emplace_back(run, i);
  run(0);
  for (auto& t : th) t.join();
  for (int i = 0; i < nplans; ++i)
    if (rcs[(size_t)i]) return sscg_fail(rcs[(size_t)i], "group rank %d: %s", i, errs[(size_t)i].c_str());
  return SSCG_OK;
}

// ---- Hestenes-Stiefel CG (classic.py:33-104) ----------------------------------
namespace {
constexpr int HS_CHUNK = 16;          // iterations per graph replay
constexpr int64_t HS_LOG_CAP = 1 << 20;  // device log rows (iterations past it are not logged)
}  // namespace

namespace {
// one HSCG iteration on the plan's stream: [halo of p and x] -> ap (+ the true
// residual) -> [allreduce p.ap, ||b-Ax||^2, ||b-Ax-r||^2] -> loop top, x, r ->
// [allreduce r.r] -> beta, p.  Two allreduces and one halo per iteration, the
// distributed classic CG of classic.py:33-104.
int hscg_capture_iter(sscg_plan* p, const Ctx& c, double* P, double* AP, double* R, bool prod) {
  if (p->partitioned && p->comm) {
    TRY(halo_exchange(p->halo, c, p->comm, p->stream));
    halo_unpack(p->halo, c, p->stream);
  }
  launch_hscg_ap(c, P, AP, R, !prod, p->stream);
  TRY(nccl_allreduce(p->comm, c.red_buf, 3, p->stream));
  launch_hscg_xr(c, P, AP, R, prod, p->stream);
  TRY(nccl_allreduce(p->comm, c.red_buf + 3, 1, p->stream));
  launch_hscg_p(c, P, R, p->stream);
  return SSCG_OK;
}
}  // namespace

int sscg_hscg_ex(sscg_plan* p, const double* b, const double* x0, double eps_star,
                 int64_t max_iters, int32_t mode, double* x_out, sscg_logs* logs) {
  if (!p || !b) return sscg_fail(SSCG_EINVAL, "NULL argument");
  if (!(eps_star >= 0.0)) return sscg_fail(SSCG_EINVAL, "eps_star must be >= 0");
  if (mode != SSCG_HSCG_REFERENCE && mode != SSCG_HSCG_PRODUCTION)
    return sscg_fail(SSCG_EINVAL, "unknown HSCG mode %d", mode);
  if (p->partitioned && !p->comm)
    return sscg_fail(SSCG_EINVAL, "a virtual-group member runs HSCG through sscg_vgroup_hscg");
  const bool prod = mode == SSCG_HSCG_PRODUCTION;
  if (max_iters < 0) max_iters = 100 * p->n;  // classic.py:46-47 (partitioned: owned rows' share)
  CUDA_OK(cudaSetDevice(p->device));
  TRY(sscg_load(p, b, x0));
  TRY(ensure_work(p, 1, std::min<int64_t>(max_iters, HS_LOG_CAP), 2));  // Y: p, ap, r
  DevConfig dc;
  memset(&dc, 0, sizeof(dc));
  dc.sigma = 1;
  dc.eps_star = eps_star;
  dc.unit = std::ldexp(1.0, -53);
  dc.c0 = sscg_host_c0();
  dc.cap_iters = p->cap_iters;
  dc.cap_outer = p->cap_outer - 1;
  dc.max_iters = max_iters;
  CUDA_OK(cudaMemcpyAsync(p->d_cfg, &dc, sizeof(dc), cudaMemcpyHostToDevice, p->stream));
  CUDA_OK(cudaMemsetAsync(p->d_it, 0xff, sizeof(double) * p->cap_iters * SSCG_IT_N, p->stream));
  p->halo.r_col = 2;  // the halo carries p (Y column 0), r (column 2) and x
  const Ctx c = make_ctx(p);
  double* P = p->d_Y;
  double* AP = p->d_Y + p->ld;
  double* R = p->d_Y + 2 * p->ld;
  if (!p->hs_gexec || p->hs_y != p->d_Y || p->hs_it != p->d_it || p->hs_mode != mode) {
    if (p->hs_gexec) cudaGraphExecDestroy(p->hs_gexec);
    p->hs_gexec = nullptr;
    cudaGraph_t g = nullptr;
    long long ar0, halo0, ar1, halo1;
    collective_counts(&ar0, &halo0);
    CUDA_OK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
    int crc = SSCG_OK;
    for (int i = 0; i < HS_CHUNK && crc == SSCG_OK; ++i) crc = hscg_capture_iter(p, c, P, AP, R, prod);
    const cudaError_t ee = cudaStreamEndCapture(p->stream, &g);
    if (crc != SSCG_OK) {
      if (g) cudaGraphDestroy(g);
      return crc;
    }
    if (ee != cudaSuccess) return sscg_fail_cuda(ee, "cudaStreamEndCapture (hscg)");
    // census per iteration of the HS_CHUNK-iteration graph
    collective_counts(&ar1, &halo1);
    graph_census(g, p->census);
    p->census[0] = (int)((ar1 - ar0) / HS_CHUNK);
    p->census[1] = (int)((halo1 - halo0) / HS_CHUNK);
    for (int k = 2; k < 5; ++k) p->census[k] /= HS_CHUNK;
    const cudaError_t e = cudaGraphInstantiate(&p->hs_gexec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return sscg_fail_cuda(e, "cudaGraphInstantiate (hscg)");
    p->hs_y = p->d_Y;
    p->hs_it = p->d_it;
    p->hs_mode = mode;
  }
  CUDA_OK(cudaEventRecord(p->ev_start, p->stream));
  launch_hscg_init(c, P, R, p->d_x0, p->stream);
  TRY(nccl_allreduce(p->comm, c.red_buf, 2, p->stream));  // ||b||^2, r.r
  launch_hscg_start(c, p->stream);
  CUDA_OK(cudaGetLastError());
  // replay chunks, polling `done` one chunk behind (the GPU never waits on the
  // host); one more chunk than max_iters / HS_CHUNK for the last loop top
  const int64_t chunks = max_iters / HS_CHUNK + 1;
  int chunk_id = 0;
  for (int64_t q = 0; q < chunks; ++q) {
    CUDA_OK(cudaGraphLaunch(p->hs_gexec, p->stream));
    const int slot = chunk_id & 1;
    CUDA_OK(cudaMemcpyAsync(p->h_done + slot, &p->d_st->done, sizeof(int), cudaMemcpyDeviceToHost,
                            p->stream));
    CUDA_OK(cudaEventRecord(p->ev_chunk[slot], p->stream));
    if (chunk_id >= 1) {
      CUDA_OK(cudaEventSynchronize(p->ev_chunk[slot ^ 1]));
      if (p->h_done[slot ^ 1]) break;
    }
    ++chunk_id;
  }
  if (prod) {  // the final x's true residual for the last trace row
    if (p->partitioned && p->comm) {
      TRY(halo_exchange(p->halo, c, p->comm, p->stream));
      halo_unpack(p->halo, c, p->stream);
    }
    launch_hscg_final(c, R, p->stream);
    TRY(nccl_allreduce(p->comm, c.red_buf + 1, 2, p->stream));
    launch_hscg_final_row(c, p->stream);
  }
  CUDA_OK(cudaEventRecord(p->ev_stop, p->stream));
  CUDA_OK(cudaStreamSynchronize(p->stream));
  CUDA_OK(cudaGetLastError());
  float ms = 0.f;
  CUDA_OK(cudaEventElapsedTime(&ms, p->ev_start, p->ev_stop));
  p->last_ms = ms;
  if (x_out) TRY(copy_d2h(p, x_out, p->d_x, sizeof(double) * p->n_own));
  if (logs) {
    SolverState st;
    CUDA_OK(cudaMemcpy(&st, p->d_st, sizeof(st), cudaMemcpyDeviceToHost));
    logs->status = st.done ? st.status : SSCG_EXHAUSTED;
    logs->total_iters = st.total_iters;
    logs->total_outer = st.total_iters;
    logs->n_records = 0;
    logs->outer_launched = chunk_id + 1;
    logs->device_ms = ms;
    const int64_t ni = std::min<int64_t>({(int64_t)st.total_iters, logs->cap_iters, p->cap_iters});
    if (logs->iters && ni > 0)
      CUDA_OK(cudaMemcpy(logs->iters, p->d_it, sizeof(double) * ni * SSCG_IT_N, cudaMemcpyDeviceToHost));
  }
  return SSCG_OK;
}

int sscg_hscg(sscg_plan* p, const double* b, const double* x0, double eps_star, int64_t max_iters,
              double* x_out, sscg_logs* logs) {
  return sscg_hscg_ex(p, b, x0, eps_star, max_iters, SSCG_HSCG_REFERENCE, x_out, logs);
}

// ---- virtual-group HSCG (single process, lock step, no NCCL) ------------------
int sscg_vgroup_hscg(sscg_plan* const* plans, int32_t np, const double* const* b,
                     const double* const* x0, double eps_star, int64_t max_iters, int32_t mode,
                     sscg_logs* logs0) {
  if (!plans || np < 1 || !b) return sscg_fail(SSCG_EINVAL, "bad group arguments");
  if (mode != SSCG_HSCG_REFERENCE && mode != SSCG_HSCG_PRODUCTION)
    return sscg_fail(SSCG_EINVAL, "unknown HSCG mode %d", mode);
  for (int i = 0; i < np; ++i)
    if (!plans[i] || !plans[i]->partitioned || plans[i]->comm || plans[i]->world != np ||
        plans[i]->rank != i || plans[i]->device != plans[0]->device)
      return sscg_fail(SSCG_EINVAL, "plan %d is not member %d of a %d-plan virtual group on one device",
                       i, i, np);
  const bool prod = mode == SSCG_HSCG_PRODUCTION;
  if (!(eps_star >= 0.0)) return sscg_fail(SSCG_EINVAL, "eps_star must be >= 0");
  if (max_iters < 0) {
    int64_t n = 0;
    for (int i = 0; i < np; ++i) n += plans[i]->n_own;
    max_iters = 100 * n;
  }
  CUDA_OK(cudaSetDevice(plans[0]->device));
  std::vector<Ctx> cs;
  std::vector<double*> reds;
  for (int i = 0; i < np; ++i) {
    sscg_plan* p = plans[i];
    TRY(sscg_load(p, b[i], x0 ? x0[i] : nullptr));
    CUDA_OK(cudaStreamSynchronize(p->stream));
    TRY(ensure_work(p, 1, std::min<int64_t>(max_iters, HS_LOG_CAP), 2));
    DevConfig dc;
    memset(&dc, 0, sizeof(dc));
    dc.sigma = 1;
    dc.eps_star = eps_star;
    dc.unit = std::ldexp(1.0, -53);
    dc.c0 = sscg_host_c0();
    dc.cap_iters = p->cap_iters;
    dc.cap_outer = p->cap_outer - 1;
    dc.max_iters = max_iters;
    CUDA_OK(cudaMemcpy(p->d_cfg, &dc, sizeof(dc), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemset(p->d_it, 0xff, sizeof(double) * p->cap_iters * SSCG_IT_N));
    p->halo.r_col = 2;
    cs.push_back(make_ctx(p));
    reds.push_back(p->d_red);
  }
  cudaStream_t s = plans[0]->stream;
  double** d_reds = nullptr;
  CUDA_OK(cudaMalloc(&d_reds, sizeof(double*) * np));
  CUDA_OK(cudaMemcpy(d_reds, reds.data(), sizeof(double*) * np, cudaMemcpyHostToDevice));
  auto Y = [&](int i, int col) { return plans[i]->d_Y + (int64_t)col * plans[i]->ld; };
  auto halo = [&]() -> int {  // pack on every member, device copies peer -> peer, unpack
    for (int i = 0; i < np; ++i) TRY(halo_exchange(plans[i]->halo, cs[i], nullptr, s));
    for (int i = 0; i < np; ++i) {
      const HaloPlan& h = plans[i]->halo;
      for (int q = 0; q < h.n_peers; ++q) {
        const int j = h.peer_rank[q];
        const HaloPlan& hj = plans[j]->halo;
        int qi = -1;
        for (int t = 0; t < hj.n_peers; ++t)
          if (hj.peer_rank[t] == i) qi = t;
        const int64_t n = h.recv_off[q + 1] - h.recv_off[q];
        if (qi < 0 || hj.send_off[qi + 1] - hj.send_off[qi] != n)
          return sscg_fail(SSCG_EINVAL, "halo lists of members %d and %d disagree", i, j);
        if (n)
          CUDA_OK(cudaMemcpyAsync(h.d_recvbuf + 3 * h.recv_off[q], hj.d_sendbuf + 3 * hj.send_off[qi],
                                  sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
      }
    }
    for (int i = 0; i < np; ++i) halo_unpack(plans[i]->halo, cs[i], s);
    return SSCG_OK;
  };
  int rc = SSCG_OK;
  for (int i = 0; i < np; ++i) launch_hscg_init(cs[i], Y(i, 0), Y(i, 2), plans[i]->d_x0, s);
  launch_vsum(d_reds, np, 2, s);
  for (int i = 0; i < np; ++i) launch_hscg_start(cs[i], s);
  int64_t it = 0;
  for (; it <= max_iters && rc == SSCG_OK; ++it) {
    rc = halo();
    if (rc) break;
    for (int i = 0; i < np; ++i) launch_hscg_ap(cs[i], Y(i, 0), Y(i, 1), Y(i, 2), !prod, s);
    launch_vsum(d_reds, np, 3, s);
    for (int i = 0; i < np; ++i) launch_hscg_xr(cs[i], Y(i, 0), Y(i, 1), Y(i, 2), prod, s);
    // the r.r slot alone (slot 3): sum in place on offset pointers
    for (int i = 0; i < np; ++i) reds[i] = plans[i]->d_red + 3;
    CUDA_OK(cudaMemcpyAsync(d_reds, reds.data(), sizeof(double*) * np, cudaMemcpyHostToDevice, s));
    launch_vsum(d_reds, np, 1, s);
    for (int i = 0; i < np; ++i) reds[i] = plans[i]->d_red;
    CUDA_OK(cudaMemcpyAsync(d_reds, reds.data(), sizeof(double*) * np, cudaMemcpyHostToDevice, s));
    for (int i = 0; i < np; ++i) launch_hscg_p(cs[i], Y(i, 0), Y(i, 2), s);
    if (it % HS_CHUNK == HS_CHUNK - 1 || it == max_iters) {
      cudaError_t e = cudaMemcpyAsync(plans[0]->h_done, &plans[0]->d_st->done, sizeof(int),
                                      cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) {
        rc = sscg_fail_cuda(e, "virtual group HSCG step");
        break;
      }
      if (plans[0]->h_done[0]) break;
    }
  }
  if (rc == SSCG_OK && prod) {
    rc = halo();
    if (rc == SSCG_OK) {
      for (int i = 0; i < np; ++i) launch_hscg_final(cs[i], Y(i, 2), s);
      for (int i = 0; i < np; ++i) reds[i] = plans[i]->d_red + 1;
      cudaMemcpyAsync(d_reds, reds.data(), sizeof(double*) * np, cudaMemcpyHostToDevice, s);
      launch_vsum(d_reds, np, 2, s);
      for (int i = 0; i < np; ++i) launch_hscg_final_row(cs[i], s);
    }
  }
  CUDA_OK(cudaStreamSynchronize(s));
  cudaFree(d_reds);
  if (rc) return rc;
  CUDA_OK(cudaGetLastError());
  if (logs0) {
    sscg_plan* p = plans[0];
    SolverState st;
    CUDA_OK(cudaMemcpy(&st, p->d_st, sizeof(st), cudaMemcpyDeviceToHost));
    logs0->status = st.done ? st.status : SSCG_EXHAUSTED;
    logs0->total_iters = st.total_iters;
    logs0->total_outer = st.total_iters;
    logs0->n_records = 0;
    const int64_t ni = std::min<int64_t>({(int64_t)st.total_iters, logs0->cap_iters, p->cap_iters});
    if (logs0->iters && ni > 0)
      CUDA_OK(cudaMemcpy(logs0->iters, p->d_it, sizeof(double) * ni * SSCG_IT_N, cudaMemcpyDeviceToHost));
  }
  return SSCG_OK;
}

// ---- power iteration (matio.py:229-244) --------------------------------------
int sscg_power_iteration(sscg_plan* p, int32_t mode, double shift, const double* v0, int32_t iters,
                         double tol, double* lam_out, int32_t* iters_used, int32_t* converged) {
  if (!p || !v0 || !lam_out) return sscg_fail(SSCG_EINVAL, "NULL argument");
  if (p->partitioned) return sscg_fail(SSCG_EINVAL, "power iteration runs on single-GPU plans");
  if (mode < 0 || mode > 2) return sscg_fail(SSCG_EINVAL, "unknown power-iteration mode %d", mode);
  CUDA_OK(cudaSetDevice(p->device));
  TRY(ensure_work(p, 1, 1, 2));  // Y columns: v, w, u
  const Ctx c = make_ctx(p);
  double* V = p->d_Y;
  double* W = p->d_Y + p->ld;
  double* U = p->d_Y + 2 * p->ld;
  double* res = p->d_red;  // two scalar slots
  CUDA_OK(cudaMemcpyAsync(V, v0, sizeof(double) * p->n, cudaMemcpyHostToDevice, p->stream));
  double lam = 0.0, h[2];
  int32_t used = iters, conv = 0;
  for (int32_t it = 1; it <= iters; ++it) {
    launch_pw_apply(c, mode, shift, V, W, nullptr, res, p->stream);  // w = op(v), w.w
    CUDA_OK(cudaMemcpyAsync(h, res, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CUDA_OK(cudaStreamSynchronize(p->stream));
    const double nw = std::sqrt(h[0]);  // np.linalg.norm of a vector: sqrt(dot(w, w))
    if (nw == 0.0) {
      lam = 0.0;
      used = it;
      conv = 1;
      break;
    }
    launch_pw_scale(p->n, W, nw, V, p->stream);                      // v = w / nw
    launch_pw_apply(c, mode, shift, V, U, V, res + 1, p->stream);    // v . op(v)
    CUDA_OK(cudaMemcpyAsync(h + 1, res + 1, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CUDA_OK(cudaStreamSynchronize(p->stream));
    const double nl = h[1];
    if (lam != 0.0 && std::fabs(nl - lam) <= tol * std::fabs(nl)) {
      lam = nl;
      used = it;
      conv = 1;
      break;
    }
    lam = nl;
  }
  CUDA_OK(cudaGetLastError());
  *lam_out = lam;
  if (iters_used) *iters_used = used;
  if (converged) *converged = conv;
  return SSCG_OK;
}

// ---- virtual-rank group (single process, lock step, no NCCL) ------------------
int sscg_vgroup_run(sscg_plan* const* plans, int32_t np, const sscg_config* cfg,
                    const double* const* b, const double* const* x0, sscg_logs* logs0) {
  if (!plans || np < 1 || !b) return sscg_fail(SSCG_EINVAL, "bad group arguments");
  for (int i = 0; i < np; ++i) {
    if (!plans[i] || !plans[i]->partitioned || plans[i]->comm || plans[i]->world != np ||
        plans[i]->rank != i || plans[i]->device != plans[0]->device)
      return sscg_fail(SSCG_EINVAL, "plan %d is not member %d of a %d-plan virtual group on one device",
                       i, i, np);
    TRY(sscg_load(plans[i], b[i], x0 ? x0[i] : nullptr));
    CUDA_OK(cudaStreamSynchronize(plans[i]->stream));
  }
  for (int i = 0; i < np; ++i) TRY(run_prepare(plans[i], cfg));
  for (int i = 0; i < np; ++i) CUDA_OK(cudaStreamSynchronize(plans[i]->stream));
  cudaStream_t s = plans[0]->stream;
  std::vector<Ctx> cs;
  std::vector<double*> reds;
  for (int i = 0; i < np; ++i) {
    cs.push_back(make_ctx(plans[i]));
    reds.push_back(plans[i]->d_red);
  }
  double** d_reds = nullptr;
  CUDA_OK(cudaMalloc(&d_reds, sizeof(double*) * np));
  CUDA_OK(cudaMemcpy(d_reds, reds.data(), sizeof(double*) * np, cudaMemcpyHostToDevice));
  const int sigma = cfg->sigma, k = 2 * sigma + 1;
  const int npack = k * (k + 1) / 2 + 2;
  for (int i = 0; i < np; ++i) {
    launch_init_residual(cs[i], plans[i]->d_x0, s);
    launch_norm_pack(cs[i], s);
  }
  launch_vsum(d_reds, np, 1, s);
  for (int i = 0; i < np; ++i) launch_state_init(cs[i], s);
  int rc = SSCG_OK;
  int launched = 0;
  for (int outer = 0; outer <= cfg->max_outer && !rc; ++outer) {
    // halo: pack on every member, device copies peer -> peer, unpack
    for (int i = 0; i < np && !rc; ++i) rc = halo_exchange(plans[i]->halo, cs[i], nullptr, s);
    for (int i = 0; i < np && !rc; ++i) {
      const HaloPlan& h = plans[i]->halo;
      for (int q = 0; q < h.n_peers && !rc; ++q) {
        const int j = h.peer_rank[q];
        const HaloPlan& hj = plans[j]->halo;
        int qi = -1;
        for (int t = 0; t < hj.n_peers; ++t)
          if (hj.peer_rank[t] == i) qi = t;
        const int64_t n = h.recv_off[q + 1] - h.recv_off[q];
        if (qi < 0 || hj.send_off[qi + 1] - hj.send_off[qi] != n) {
          rc = sscg_fail(SSCG_EINVAL, "halo lists of members %d and %d disagree", i, j);
          break;
        }
        if (n) {
          cudaError_t e = cudaMemcpyAsync(h.d_recvbuf + 3 * h.recv_off[q], hj.d_sendbuf + 3 * hj.send_off[qi],
                                          sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s);
          if (e != cudaSuccess) rc = sscg_fail_cuda(e, "halo copy");
        }
      }
    }
    if (rc) break;
    for (int i = 0; i < np; ++i) halo_unpack(plans[i]->halo, cs[i], s);
    for (int i = 0; i < np; ++i) {
      launch_params_begin(cs[i], s);
      for (int n = 2; n < sigma; ++n) launch_leja_point(cs[i], n, s);
      for (int l = 0; l < sigma; ++l) launch_level(cs[i], l, sigma, s);
      launch_gram(cs[i], k, s);
    }
    launch_vsum(d_reds, np, npack, s);
    for (int i = 0; i < np; ++i) {
      launch_small(cs[i], s);
      launch_recover(cs[i], s);
    }
    ++launched;
    int done = 0;
    cudaError_t e = cudaMemcpyAsync(plans[0]->h_done, &plans[0]->d_st->done, sizeof(int),
                                    cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      rc = sscg_fail_cuda(e, "virtual group step");
      break;
    }
    done = plans[0]->h_done[0];
    if (done) break;
  }
  cudaFree(d_reds);
  if (rc) return rc;
  CUDA_OK(cudaGetLastError());
  for (int i = 0; i < np; ++i) plans[i]->last_launched = launched;
  if (logs0) TRY(sscg_fetch(plans[0], nullptr, logs0));
  return SSCG_OK;
}

// ---- unit entry points ------------------------------------------------------
int sscg_spmv(sscg_plan* p, const double* x, double* y) {
  if (!p || !x || !y) return sscg_fail(SSCG_EINVAL, "NULL argument");
  CUDA_OK(cudaSetDevice(p->device));
  CUDA_OK(cudaMemcpyAsync(p->d_xj, x, sizeof(double) * p->n, cudaMemcpyHostToDevice, p->stream));
  launch_spmv(p->d_rp, p->d_col, p->d_val, p->n, p->d_xj, p->d_rj, p->stream);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaMemcpyAsync(y, p->d_rj, sizeof(double) * p->n, cudaMemcpyDeviceToHost, p->stream));
  CUDA_OK(cudaStreamSynchronize(p->stream));
  return SSCG_OK;
}

int sscg_build_block(sscg_plan* p, const double* pv, const double* rv, int32_t s,
                     const double* th, const double* ga, const double* mu, double* y_out,
                     double* g_out) {
  if (!p || !pv || !rv || !th || !ga || (s > 1 && !mu)) return sscg_fail(SSCG_EINVAL, "NULL argument");
  if (s < 1 || s > SMAX) return sscg_fail(SSCG_EINVAL, "s=%d outside [1, %d]", s, SMAX);
  CUDA_OK(cudaSetDevice(p->device));
  const int k = 2 * s + 1;
  double *dY = nullptr, *part = nullptr, *dg = nullptr;
  int* flag = nullptr;
  int rc = SSCG_OK;
  cudaError_t e = cudaSuccess;
  int h_flag = 0;
  if ((e = cudaMalloc(&dY, sizeof(double) * p->ld * k)) || (e = cudaMalloc(&part, sizeof(double) * GRAM_BLOCKS * GPACK)) ||
      (e = cudaMalloc(&dg, sizeof(double) * k * k)) || (e = cudaMalloc(&flag, 2 * sizeof(int))) ||
      (e = cudaMemset(dY, 0, sizeof(double) * p->ld * k)) || (e = cudaMemset(flag, 0, 2 * sizeof(int))) ||
      (e = cudaMemcpy(dY, pv, sizeof(double) * p->n, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(dY + (size_t)(s + 1) * p->ld, rv, sizeof(double) * p->n, cudaMemcpyHostToDevice))) {
    rc = sscg_fail_cuda(e, "build_block setup");
  } else {
    launch_block_levels(p->d_rp, p->d_col, p->d_val, p->n, p->ld, dY, s, th, ga, mu, flag, p->stream);
    launch_gram_raw(dY, p->n, p->ld, k, part, dg, flag + 1, p->stream);
    if ((e = cudaStreamSynchronize(p->stream)) || (e = cudaGetLastError()) ||
        (e = cudaMemcpy(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost))) {
      rc = sscg_fail_cuda(e, "build_block");
    } else if (h_flag) {
      rc = sscg_fail(SSCG_EBREAKDOWN, "non-finite basis column (BasisBreakdownError)");
    } else {
      for (int col = 0; col < k && !rc; ++col)
        if ((e = cudaMemcpy(y_out + (size_t)col * p->n, dY + (size_t)col * p->ld, sizeof(double) * p->n,
                            cudaMemcpyDeviceToHost)))
          rc = sscg_fail_cuda(e, "download Y");
      if (!rc && g_out && (e = cudaMemcpy(g_out, dg, sizeof(double) * k * k, cudaMemcpyDeviceToHost)))
        rc = sscg_fail_cuda(e, "download G");
    }
  }
  cudaFree(dY);
  cudaFree(part);
  cudaFree(dg);
  cudaFree(flag);
  return rc;
}

int sscg_gram(int32_t device, int64_t n, int32_t k, const double* y, double* g) {
  if (!y || !g || n < 1 || k < 1 || k > CMAX) return sscg_fail(SSCG_EINVAL, "bad gram arguments");
  CUDA_OK(cudaSetDevice(device));
  const int64_t ld = round_up(n, gram_row_multiple());
  double *dY = nullptr, *part = nullptr, *dg = nullptr;
  int* cnt = nullptr;
  int rc = SSCG_OK;
  cudaError_t e;
  if ((e = cudaMalloc(&dY, sizeof(double) * ld * k)) || (e = cudaMalloc(&part, sizeof(double) * GRAM_BLOCKS * GPACK)) ||
      (e = cudaMalloc(&dg, sizeof(double) * k * k)) || (e = cudaMalloc(&cnt, sizeof(int))) ||
      (e = cudaMemset(dY, 0, sizeof(double) * ld * k)) || (e = cudaMemset(cnt, 0, sizeof(int))) ||
      (e = cudaMemcpy2D(dY, ld * sizeof(double), y, n * sizeof(double), n * sizeof(double), k,
                        cudaMemcpyHostToDevice))) {
    rc = sscg_fail_cuda(e, "gram setup");
  } else {
    launch_gram_raw(dY, n, ld, k, part, dg, cnt, 0);
    if ((e = cudaDeviceSynchronize()) || (e = cudaGetLastError()) ||
        (e = cudaMemcpy(g, dg, sizeof(double) * k * k, cudaMemcpyDeviceToHost)))
      rc = sscg_fail_cuda(e, "gram");
  }
  cudaFree(dY);
  cudaFree(part);
  cudaFree(dg);
  cudaFree(cnt);
  return rc;
}

int sscg_recover(int32_t device, int64_t n, int32_t k, const double* y, const double* xp,
                 const double* rp, const double* pp, const double* xb, double* x, double* r,
                 double* pout) {
  if (!y || !xp || !rp || !pp || !xb || !x || !r || !pout || n < 1 || k < 1 || k > CMAX)
    return sscg_fail(SSCG_EINVAL, "bad recover arguments");
  CUDA_OK(cudaSetDevice(device));
  const int64_t ld = round_up(n, 64);
  double *dY = nullptr, *coef = nullptr, *dxb = nullptr, *dx = nullptr, *dr = nullptr, *dp = nullptr;
  int rc = SSCG_OK;
  cudaError_t e;
  std::vector<double> hc(3 * k);
  for (int i = 0; i < k; ++i) {
    hc[i] = xp[i];
    hc[k + i] = rp[i];
    hc[2 * k + i] = pp[i];
  }
  if ((e = cudaMalloc(&dY, sizeof(double) * ld * k)) || (e = cudaMalloc(&coef, sizeof(double) * 3 * k)) ||
      (e = cudaMalloc(&dxb, sizeof(double) * ld)) || (e = cudaMalloc(&dx, sizeof(double) * ld)) ||
      (e = cudaMalloc(&dr, sizeof(double) * ld)) || (e = cudaMalloc(&dp, sizeof(double) * ld)) ||
      (e = cudaMemset(dY, 0, sizeof(double) * ld * k)) || (e = cudaMemset(dxb, 0, sizeof(double) * ld)) ||
      (e = cudaMemcpy2D(dY, ld * sizeof(double), y, n * sizeof(double), n * sizeof(double), k,
                        cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(coef, hc.data(), sizeof(double) * 3 * k, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(dxb, xb, sizeof(double) * n, cudaMemcpyHostToDevice))) {
    rc = sscg_fail_cuda(e, "recover setup");
  } else {
    launch_recover_raw(dY, n, ld, k, coef, dxb, dx, dr, dp, 0);
    if ((e = cudaDeviceSynchronize()) || (e = cudaGetLastError()) ||
        (e = cudaMemcpy(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(r, dr, sizeof(double) * n, cudaMemcpyDeviceToHost)) ||
        (e = cudaMemcpy(pout, dp, sizeof(double) * n, cudaMemcpyDeviceToHost)))
      rc = sscg_fail_cuda(e, "recover");
  }
  for (double* b : {dY, coef, dxb, dx, dr, dp}) cudaFree(b);
  return rc;
}

int sscg_nested_conds(int32_t device, const double* g, int32_t s_bar, double* conds) {
  if (!g || !conds || s_bar < 1 || s_bar > SMAX) return sscg_fail(SSCG_EINVAL, "bad arguments");
  CUDA_OK(cudaSetDevice(device));
  return unit_nested_conds(g, s_bar, conds, 0, 1.0, 1.0, 1.0, 1.0, nullptr);
}

int sscg_select_s_tilde(int32_t device, const double* g, int32_t s_bar, double c, double unit,
                        double eps_star, double r_norm, int32_t* s_tilde, double* conds) {
  if (!g || !conds || !s_tilde || s_bar < 1 || s_bar > SMAX)
    return sscg_fail(SSCG_EINVAL, "bad arguments");
  CUDA_OK(cudaSetDevice(device));
  int st = 1;
  TRY(unit_nested_conds(g, s_bar, conds, 1, c, unit, eps_star, r_norm, &st));
  *s_tilde = st;
  return SSCG_OK;
}

int sscg_leja_points(int32_t device, double lmin, double lmax, int32_t count, int32_t grid,
                     double* out) {
  if (!out || count < 1 || count > SMAX || grid < 2) return sscg_fail(SSCG_EINVAL, "bad arguments");
  if (!(0.0 <= lmin && lmin < lmax))
    return sscg_fail(SSCG_EPARAM, "need 0 <= lmin < lmax, got (%g, %g)", lmin, lmax);
  CUDA_OK(cudaSetDevice(device));
  return unit_leja(lmin, lmax, count, grid, out);
}

int sscg_params_for(int32_t device, int32_t kind, int32_t s, int32_t has, double lmin, double lmax,
                    int32_t grid, double* th, double* ga, double* mu, int32_t* kind_out) {
  if (kind < 0 || kind > 2) return sscg_fail(SSCG_EPARAM, "unknown basis kind %d", kind);
  if (s < 1 || s > SMAX || !th || !ga || !mu || !kind_out || grid < 2)
    return sscg_fail(SSCG_EINVAL, "bad arguments");
  CUDA_OK(cudaSetDevice(device));
  int ko = 0;
  TRY(unit_params_for(kind, s, has, lmin, lmax, grid, th, ga, mu, &ko));
  *kind_out = ko;
  return SSCG_OK;
}

int sscg_ritz_sequence(int32_t device, int32_t m, const double* alpha, const double* beta,
                       double* rec) {
  if (m < 0 || (m && (!alpha || !beta || !rec))) return sscg_fail(SSCG_EINVAL, "bad arguments");
  if (m == 0) return SSCG_OK;
  CUDA_OK(cudaSetDevice(device));
  return unit_ritz(m, alpha, beta, rec);
}

int sscg_sym_eig(int32_t device, int32_t n, const double* m, double* w) {
  if (!m || !w || n < 1 || n > CMAX) return sscg_fail(SSCG_EINVAL, "bad arguments");
  CUDA_OK(cudaSetDevice(device));
  return unit_sym_eig(n, m, w);
}

}  // extern "C"
