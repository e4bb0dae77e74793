// fp64 log and 64-bit shuffle dependent latencies on one warp (B200):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/log_probe.bin tools/log_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int iters) {
  double a = 3.0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = log(fabs(a - 1.5) + 1e-300) + 4.0;
  long long t1 = clock64();
  double b = a;
  for (int i = 0; i < iters; ++i) b = __shfl_xor_sync(0xffffffffu, b, 1) + 1.0;
  long long t2 = clock64();
  double c = b;
  for (int i = 0; i < iters; ++i) c = (c > 2.0) ? c * 0.5 : c + 1.0;
  long long t3 = clock64();
  out[threadIdx.x] = a + b + c;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 32 * 8); cudaMallocManaged(&cyc, 3 * 8);
  const int iters = 2048;
  k<<<1, 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  printf("log+2 adds: %.1f cycles; shfl64+add: %.1f; compare/select/mul: %.1f\n",
         (double)cyc[0] / iters, (double)cyc[1] / iters, (double)cyc[2] / iters);
  return 0;
}
