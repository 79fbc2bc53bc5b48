// Probe: which 4-D fp32 TMA tile loads are legal on sm_100a (box vs global dims).
// usage: tma_probe W H C N boxW boxH boxC c0 c1
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, uint32_t bytes, float* out, int n) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar)), "r"(bytes));
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      :: "r"(sa(sm)), "l"((uint64_t)&m), "r"(c0), "r"(c1), "r"(0), "r"(0), "r"(sa(&bar)) : "memory");
  }
  uint32_t done = 0;
  while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }" : "=r"(done) : "r"(sa(&bar)));
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = sm[i];
}

int main(int argc, char** argv) {
  int W = atoi(argv[1]), H = atoi(argv[2]), C = atoi(argv[3]), N = atoi(argv[4]);
  int bW = atoi(argv[5]), bH = atoi(argv[6]), bC = atoi(argv[7]), c0 = atoi(argv[8]), c1 = atoi(argv[9]);
  float* x; cudaMalloc(&x, (size_t)W * H * C * N * 4);
  std::vector<float> h((size_t)W * H * C * N); for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i + 1);
  cudaMemcpy(x, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C, (cuuint64_t)N};
  cuuint64_t st[3] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4, (cuuint64_t)W * H * C * 4};
  cuuint32_t box[4] = {(cuuint32_t)bW, (cuuint32_t)bH, (cuuint32_t)bC, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int n = bW * bH * bC; float* out; cudaMalloc(&out, n * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<1, 128, n * 4>>>(m, c0, c1, (uint32_t)n * 4, out, n);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> o(n); cudaMemcpy(o.data(), out, n * 4, cudaMemcpyDeviceToHost);
  printf("W=%d H=%d C=%d box=%dx%dx%d at (%d,%d): encode=%d kernel=%s first=%g %g %g\n", W, H, C, bW, bH, bC, c0, c1,
         (int)r, cudaGetErrorString(e), o[0], o[1], o[2]);
  return 0;
}
