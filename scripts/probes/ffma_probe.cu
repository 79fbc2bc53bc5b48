// Probe: FP32 FFMA vs packed FFMA2 (fma.rn.f32x2) throughput on sm_100a, with and
// without interleaved integer/LDS overhead instructions.  Prints TFLOP/s.
#include <cuda_runtime.h>
#include <cstdio>

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters, float a) {
  __shared__ float sh[1024];
  sh[threadIdx.x] = threadIdx.x; __syncthreads();
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = threadIdx.x * 0.001f + i;
  float x0 = a, x1 = a * 1.5f;
  int p = threadIdx.x, q = threadIdx.x * 3, rr = threadIdx.x ^ 5, r2 = threadIdx.x + 11, q2 = threadIdx.x * 7;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = __fmaf_rn(x0, acc[i], x1);
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float2 r = __ffma2_rn(make_float2(x0, x0), make_float2(acc[i], acc[i + 1]), make_float2(x1, x1));
        acc[i] = r.x; acc[i + 1] = r.y;
      }
    } else if (MODE == 2) {  // FFMA2 + 8 overhead ops per 16 FFMA2
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        float2 r = __ffma2_rn(make_float2(x0, x0), make_float2(acc[i], acc[i + 1]), make_float2(x1, x1));
        acc[i] = r.x; acc[i + 1] = r.y;
        if ((i & 3) == 0) { asm volatile("xor.b32 %0, %0, %1;" : "+r"(p) : "r"(q)); asm volatile("add.s32 %0, %0, %1;" : "+r"(q) : "r"(rr)); asm volatile("xor.b32 %0, %0, %1;" : "+r"(r2) : "r"(q2)); asm volatile("add.s32 %0, %0, %1;" : "+r"(q2) : "r"(rr)); }
      }
    } else {  // FFMA + same overhead
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        acc[i] = __fmaf_rn(x0, acc[i], x1);
        if ((i & 3) == 0) { asm volatile("xor.b32 %0, %0, %1;" : "+r"(p) : "r"(q)); asm volatile("add.s32 %0, %0, %1;" : "+r"(q) : "r"(rr)); asm volatile("xor.b32 %0, %0, %1;" : "+r"(r2) : "r"(q2)); asm volatile("add.s32 %0, %0, %1;" : "+r"(q2) : "r"(rr)); }
      }
    }
  }
  float s = 0; for (int i = 0; i < 32; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + p + q + r2 + q2;
}

template <int MODE> void run(const char* name, int blocks, int iters) {
  float* out; cudaMalloc(&out, blocks * 256 * 4);
  k<MODE><<<blocks, 256>>>(out, 10, 1.0f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<blocks, 256>>>(out, iters, 0.999f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fl = 2.0 * 32 * iters * (double)blocks * 256;
  printf("%-28s blocks=%d %.3f ms  %.1f TFLOP/s  err=%s\n", name, blocks, ms, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int bpsm : {2, 4, 8}) {
    int blocks = 148 * bpsm;
    run<0>("ffma", blocks, 20000);
    run<1>("ffma2", blocks, 20000);
    run<3>("ffma+16 alu per 32", blocks, 20000);
    run<2>("ffma2(16)+16 alu", blocks, 20000);
  }
}
