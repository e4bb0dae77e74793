// tma_probe.cu -- standalone check of the TMA box load the plane march uses
// (4-D f64 map, 34 x 10 box with a -1 offset halo, zero fill out of bounds).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

struct Maps { CUtensorMap y; };

__global__ void k_probe(const __grid_constant__ Maps m, const CUtensorMap* gm, double* out, int c0,
                        int c1, int c2, int c3, unsigned bytes) {
  const CUtensorMap* mp = gm ? gm : &m.y;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  unsigned d0 = (unsigned)__cvta_generic_to_shared(sm);
  const int align = c3 < 0 ? 1 : 128;  // (unused)
  unsigned d = (d0 + 127u) & ~127u;
  unsigned char* smp = sm + (d - d0);
  if (threadIdx.x == 0 && blockIdx.x == 0) printf("dyn smem at 0x%x -> 0x%x, bar at 0x%x\n", d0, d, b);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(d),
        "l"(reinterpret_cast<uint64_t>(mp)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(b)
        : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(b), "r"(0u) : "memory");
  for (int i = threadIdx.x; i < 340; i += blockDim.x) out[i] = reinterpret_cast<double*>(smp)[i];
}

__global__ void k_probe2d(const __grid_constant__ CUtensorMap m, double* out, int c0, int c1) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  unsigned d = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(32 * 8 * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(d),
        "l"(reinterpret_cast<uint64_t>(&m)), "r"(c0), "r"(c1), "r"(b)
        : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(b), "r"(0u) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = reinterpret_cast<double*>(sm)[i];
}

int main(int argc, char** argv) {
  if (argc > 1 && atoi(argv[1]) == 0) {  // 2-D probe: 64 x 64 doubles, box 32 x 8 at (0, 0)
    double* a;
    cudaMalloc(&a, 64 * 64 * 8);
    std::vector<double> h(64 * 64);
    for (int i = 0; i < 64 * 64; ++i) h[i] = i;
    cudaMemcpy(a, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    double* out;
    cudaMalloc(&out, 256 * 8);
    CUtensorMap m;
    cuuint64_t dims[2] = {64, 64}, str[1] = {64 * 8};
    cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, str, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int c0 = argc > 2 ? atoi(argv[2]) : 0, c1 = argc > 3 ? atoi(argv[3]) : 0;
    k_probe2d<<<1, 128, 4096>>>(m, out, c0, c1);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> o(256);
    cudaMemcpy(o.data(), out, 256 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < 8; ++j) for (int i = 0; i < 32; ++i) { int x = c0 + i, y = c1 + j; double w = (x < 0 || y < 0) ? 0.0 : (double)(y * 64 + x); bad += o[j * 32 + i] != w; }
    printf("2-D probe: encode %d, %s, %d mismatches\n", (int)r, cudaGetErrorString(e), bad);
    return 0;
  }
  const int bw = argc > 1 ? atoi(argv[1]) : 34, bh = argc > 2 ? atoi(argv[2]) : 10;
  const int use_global = argc > 3 ? atoi(argv[3]) : 0;
  const int promo = argc > 4 ? atoi(argv[4]) : 3;
  const int o = 32, lines = 32, planes = 32, ncols = 25;
  const size_t ld = (size_t)o * lines * planes;
  std::vector<double> h(ld * ncols);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *dy, *dout;
  cudaMalloc(&dy, h.size() * 8);
  cudaMalloc(&dout, 340 * 8);
  cudaMemcpy(dy, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  if (argc > 5 && atoi(argv[5]) == 1) enc = &cuTensorMapEncodeTiled;  // the driver API directly
  Maps m;
  cuuint64_t dims[4] = {(cuuint64_t)o, (cuuint64_t)lines, (cuuint64_t)planes, (cuuint64_t)ncols};
  cuuint64_t str[3] = {8ull * o, 8ull * o * lines, 8ull * ld};
  cuuint32_t box[4] = {(cuuint32_t)bw, (cuuint32_t)bh, 1, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&m.y, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, dy, dims, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   (CUtensorMapL2promotion)promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* gm = nullptr;
  if (use_global) {
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &m.y, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  }
  printf("box %d x %d global %d promo %d: ", bw, bh, use_global, promo);
  printf("encode %d (query %d)\n", (int)r, (int)q);
  int coords[][4] = {{0, 0, 1, 2}, {2, 1, 1, 2}, {-2, 0, 1, 2}, {0, -1, 1, 2}, {-2, -1, 0, 0},
                     {-2, 7, -1, 0}, {-2, 23, 31, 24}, {30, -1, 5, 3}};
  for (auto& c : coords) {
    k_probe<<<1, 128, 340 * 8 + 256>>>(m, gm, dout, c[0], c[1], c[2], c[3], bw * bh * 8);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> out(340);
    cudaMemcpy(out.data(), dout, 340 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < bh; ++j)
      for (int i = 0; i < bw; ++i) {
        int x = c[0] + i, y = c[1] + j, z = c[2], col = c[3];
        double want = (x < 0 || x >= o || y < 0 || y >= lines || z < 0 || z >= planes) ? 0.0
                      : (double)(col * ld + (size_t)z * o * lines + (size_t)y * o + x);
        bad += out[j * bw + i] != want;
      }
    printf("coords %d %d %d %d: %s, %d mismatches\n", c[0], c[1], c[2], c[3], cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
