// rec.cu -- K_rec: fused basis recovery  x <- x + Y x',  r <- Y r',  p <- Y p'.
//
// Reference: adaptive.py:249-251 (three OpenBLAS dgemv over the copied Y_t) and
// sstep.py:37-44 `recover_iterates`.  One streaming pass reads the 2 s~ + 1 active
// columns of Y (P_0..P_s~, R_0..R_{s~-1}: no Y_t copy) and x once and writes
// x, r, p; r and p go straight back into Y's columns sigma+1 and 0 (each thread
// owns its rows, so in place is safe).  Two rows per thread, 16-byte accesses.
//
// Roofline: HBM-bound, 8 n (2 s~ + 1) + 8 n read + 24 n written per outer loop.
#include "internal.cuh"

namespace {

constexpr int REC_THREADS = 256;
#ifndef REC_UNROLL  // column loads in flight per thread (c5w full solve: 0.83 -> 0.72 ms)
#define REC_UNROLL 4
#endif
constexpr int kRecUnroll = REC_UNROLL;

// rows recovery updates: single GPU the whole padded column (padding stays 0);
// row-partitioned: the owned rows (ghosts are refreshed by the next exchange)
__device__ __forceinline__ int64_t rec_rows(const Ctx& c) {
  return c.n_own == c.n ? c.ld : ((c.n_own + 1) & ~(int64_t)1);
}

struct ColSet {
  int n;
  int col[CMAX];
};

// active physical columns in reference order (adaptive.py:107-108)
__device__ __forceinline__ void active_cols(int s_t, int sigma, int* cols) {
  for (int i = 0; i <= s_t; ++i) cols[i] = i;
  for (int i = 0; i < s_t; ++i) cols[s_t + 1 + i] = sigma + 1 + i;
}

template <bool WITH_P>
__device__ __forceinline__ void combine(const double* __restrict__ Y, int64_t ld, int64_t i2,
                                        int k, const int* cols, const double* cx,
                                        const double* cr, const double* cp, double2& sx,
                                        double2& sr, double2& sp) {
  sx = make_double2(0.0, 0.0);
  sr = sx;
  sp = sx;
#pragma unroll kRecUnroll
  for (int q = 0; q < k; ++q) {
    const int cc = cols[q];
    const double2 y = *reinterpret_cast<const double2*>(Y + (int64_t)cc * ld + i2);
    const double a = cx[cc], b = cr[cc];
    sx.x = fma(y.x, a, sx.x);
    sx.y = fma(y.y, a, sx.y);
    sr.x = fma(y.x, b, sr.x);
    sr.y = fma(y.y, b, sr.y);
    if (WITH_P) {
      const double c = cp[cc];
      sp.x = fma(y.x, c, sp.x);
      sp.y = fma(y.y, c, sp.y);
    }
  }
}

__global__ void __launch_bounds__(REC_THREADS) k_recover(Ctx c) {
  __shared__ double sx_[CMAX], sr_[CMAX], sp_[CMAX];
  __shared__ int cols[CMAX];
  const SolverState* st = c.st;
  if (!st->rec_valid) return;
  TL_K(c, -1);
  TL_BEGIN(c, 18);
  const int sigma = c.cfg->sigma, s_t = st->s_tilde;
  const int k = 2 * s_t + 1;
  if (threadIdx.x == 0) active_cols(s_t, sigma, cols);
  if (threadIdx.x < CMAX) {
    sx_[threadIdx.x] = st->cx[threadIdx.x];
    sr_[threadIdx.x] = st->cr[threadIdx.x];
    sp_[threadIdx.x] = st->cp[threadIdx.x];
  }
  __syncthreads();
  double* P0 = c.Y;
  double* R0 = c.Y + (int64_t)(sigma + 1) * c.ld;
  const int64_t lim = rec_rows(c);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
  for (int64_t i2 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; i2 < lim; i2 += stride) {
    double2 ax, ar, ap;
    combine<true>(c.Y, c.ld, i2, k, cols, sx_, sr_, sp_, ax, ar, ap);
    double2 xv = *reinterpret_cast<const double2*>(c.x + i2);
    xv.x = __dadd_rn(xv.x, ax.x);
    xv.y = __dadd_rn(xv.y, ax.y);
    *reinterpret_cast<double2*>(c.x + i2) = xv;
    *reinterpret_cast<double2*>(R0 + i2) = ar;
    *reinterpret_cast<double2*>(P0 + i2) = ap;
  }
  TL_END(c, 18);
}

// full trace: x_j = x + Y x'_j, r_j = Y r'_j into scratch (adaptive.py:205)
__global__ void __launch_bounds__(REC_THREADS) k_diag_form(Ctx c, int j) {
  __shared__ double sx_[CMAX], sr_[CMAX];
  __shared__ int cols[CMAX];
  const SolverState* st = c.st;
  if (j >= st->diag_n) return;
  const int sigma = c.cfg->sigma, s_t = st->s_tilde;
  const int k = 2 * s_t + 1;
  if (threadIdx.x == 0) active_cols(s_t, sigma, cols);
  if (threadIdx.x < CMAX) {
    sx_[threadIdx.x] = st->dx[j][threadIdx.x];
    sr_[threadIdx.x] = st->dr[j][threadIdx.x];
  }
  __syncthreads();
  const int64_t lim = rec_rows(c);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
  for (int64_t i2 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; i2 < lim; i2 += stride) {
    double2 ax, ar, ap;
    combine<false>(c.Y, c.ld, i2, k, cols, sx_, sr_, nullptr, ax, ar, ap);
    double2 xv = *reinterpret_cast<const double2*>(c.x + i2);
    xv.x = __dadd_rn(xv.x, ax.x);
    xv.y = __dadd_rn(xv.y, ax.y);
    *reinterpret_cast<double2*>(c.xj + i2) = xv;
    *reinterpret_cast<double2*>(c.rj + i2) = ar;
  }
}

// unit entry: Y has k contiguous columns; coef = [xp | rp | pp] (3 k)
__global__ void __launch_bounds__(REC_THREADS)
    k_recover_raw(const double* __restrict__ Y, int64_t ld, int k, const double* coef,
                  const double* xbase, double* x, double* r, double* p) {
  __shared__ double sx_[CMAX], sr_[CMAX], sp_[CMAX];
  __shared__ int cols[CMAX];
  if (threadIdx.x < k) {
    sx_[threadIdx.x] = coef[threadIdx.x];
    sr_[threadIdx.x] = coef[k + threadIdx.x];
    sp_[threadIdx.x] = coef[2 * k + threadIdx.x];
    cols[threadIdx.x] = threadIdx.x;
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
  for (int64_t i2 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; i2 < ld; i2 += stride) {
    double2 ax, ar, ap;
    combine<true>(Y, ld, i2, k, cols, sx_, sr_, sp_, ax, ar, ap);
    double2 xv = *reinterpret_cast<const double2*>(xbase + i2);
    xv.x = __dadd_rn(xv.x, ax.x);
    xv.y = __dadd_rn(xv.y, ax.y);
    *reinterpret_cast<double2*>(x + i2) = xv;
    *reinterpret_cast<double2*>(r + i2) = ar;
    *reinterpret_cast<double2*>(p + i2) = ap;
  }
}

// one full wave of resident CTAs (grid-stride loops): a partial second wave
// would leave most SMs idle at the tail of this HBM-bound pass
int rec_grid(int64_t ld) {
  // occupancy and SM count per device (a process may drive several GPUs)
  static std::atomic<int> cache_sms[64], cache_per_sm[64];
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  int sms = cache_sms[dev].load(std::memory_order_relaxed);
  int per_sm = cache_per_sm[dev].load(std::memory_order_relaxed);
  if (!per_sm) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_recover, REC_THREADS, 0);
    if (per_sm < 1) per_sm = 1;
    cache_sms[dev].store(sms, std::memory_order_relaxed);
    cache_per_sm[dev].store(per_sm, std::memory_order_relaxed);
  }
  int64_t g = (ld / 2 + REC_THREADS - 1) / REC_THREADS;
#ifdef REC_PER_SM
  const int64_t cap = (int64_t)sms * REC_PER_SM;
#else
  const int64_t cap = (int64_t)sms * per_sm;
#endif
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

void launch_recover(const Ctx& c, cudaStream_t s) {
  k_recover<<<rec_grid(c.ld), REC_THREADS, 0, s>>>(c);
}
void launch_diag_form(const Ctx& c, int j, cudaStream_t s) {
  k_diag_form<<<rec_grid(c.ld), REC_THREADS, 0, s>>>(c, j);
}
void launch_recover_raw(const double* Y, int64_t n, int64_t ld, int k, const double* coef,
                        const double* xbase, double* x, double* r, double* p, cudaStream_t s) {
  (void)n;
  k_recover_raw<<<rec_grid(ld), REC_THREADS, 0, s>>>(Y, ld, k, coef, xbase, x, r, p);
}
