// DFMA dependent-issue latency and per-SMSP throughput on one SM (B200):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dfma_probe.bin tools/dfma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int chains, int iters) {
  double a[8];
  for (int c = 0; c < 8; ++c) a[c] = 1.0 + threadIdx.x * 1e-9 + c;
  const double m = 1.0000001, b = 1e-9;
  __syncthreads();
  const long long t0 = clock64();
  if (chains == 1) {
    for (int i = 0; i < iters; ++i) a[0] = fma(a[0], m, b);
  } else if (chains == 2) {
    for (int i = 0; i < iters; ++i) { a[0] = fma(a[0], m, b); a[1] = fma(a[1], m, b); }
  } else if (chains == 4) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < 4; ++c) a[c] = fma(a[c], m, b);
    }
  } else {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int c = 0; c < 8; ++c) a[c] = fma(a[c], m, b);
    }
  }
  const long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < 8; ++c) s += a[c];
  out[threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 32 * 8);
  const int iters = 4096;
  for (int warps : {1, 4, 8, 16}) for (int chains : {1, 2, 4, 8}) {
    k<<<1, warps * 32>>>(out, cyc, chains, iters);
    cudaDeviceSynchronize();
    printf("warps=%2d chains=%d: %.1f cycles per loop iteration (%.2f per DFMA warp-instr per SMSP-warp)\n",
           warps, chains, (double)cyc[0] / iters, (double)cyc[0] / iters / chains);
  }
  return 0;
}
