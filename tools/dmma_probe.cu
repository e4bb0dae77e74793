// fp64 tensor-core shapes on sm_100a: which mma.sync f64 shapes assemble, what
// SASS they become and the rate each sustains (one CTA of 8 warps per SM slot,
// 4 independent accumulator sets per warp).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dmma_probe.bin tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void __launch_bounds__(256) k_probe(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + threadIdx.x * 1e-9 + i;
  double c[4][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (SHAPE == 0) {  // m8n8k4
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a[u]), "d"(b[u]));
      } else if (SHAPE == 1) {  // m16n8k4
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
                     : "d"(a[u]), "d"(a[u + 4]), "d"(b[u]));
      } else if (SHAPE == 2) {  // m16n8k8
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else {  // m16n8k16
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double s = 0;
  for (int u = 0; u < 4; ++u) for (int i = 0; i < 4; ++i) s += c[u][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SHAPE>
void run(const char* name, double macs_per_mma, int ctas_per_sm) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * ctas_per_sm, iters = 20000;
  double* out;
  cudaMalloc(&out, sizeof(double) * grid * 256);
  k_probe<SHAPE><<<grid, 256>>>(out, 100);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_probe<SHAPE><<<grid, 256>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double mmas = (double)grid * 8 * iters * 4;
  printf("%-10s ctas/SM %d  %.3f ms  %.2f TFLOP/s  (%s)\n", name, ctas_per_sm, ms,
         2.0 * mmas * macs_per_mma / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int c = 1; c <= 2; ++c) {
    run<0>("m8n8k4", 8 * 8 * 4, c);
    run<1>("m16n8k4", 16 * 8 * 4, c);
    run<2>("m16n8k8", 16 * 8 * 8, c);
    run<3>("m16n8k16", 16 * 8 * 16, c);
  }
  return 0;
}
