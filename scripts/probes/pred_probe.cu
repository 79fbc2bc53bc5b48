// Probe: does a predicated-off FFMA2 cost only an issue slot, or also FMA-pipe time?
// 32 independent FFMA2 per iteration; predicate true for `on` of every 8 instructions
// (warp-uniform).  Reports useful TFLOP/s and instruction rate.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int ON>
__global__ void __launch_bounds__(256, 1) k(float* out, int iters, uint32_t mask, uint64_t a, uint64_t b) {
  uint64_t acc[32];
  for (int i = 0; i < 32; ++i) acc[i] = (uint64_t)(threadIdx.x + i) * 0x3f8000003f800000ull;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      // predicate bit i%8 of mask (uniform); ON of 8 set
      asm volatile("{ .reg .pred p; .reg .b32 t; and.b32 t, %3, %4; setp.ne.u32 p, t, 0;"
                   " @p fma.rn.f32x2 %0, %1, %2, %0; }"
                   : "+l"(acc[i]) : "l"(a), "l"(b), "r"(mask), "r"(1u << (i % 8)));
    }
    mask = (mask << 1) | (mask >> 7);  // rotate so the compiler cannot fold
    mask &= 0xff;
  }
  float s = 0; for (int i = 0; i < 32; ++i) s += __uint_as_float((uint32_t)acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ON> void run(uint32_t mask) {
  const int blocks = 148 * 2, iters = 20000;
  float* out; cudaMalloc(&out, blocks * 256 * 4);
  k<ON><<<blocks, 256>>>(out, 10, mask, 0x3f8123453f812345ull, 0x3f7fff013f7fff01ull);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<ON><<<blocks, 256>>>(out, iters, mask, 0x3f8123453f812345ull, 0x3f7fff013f7fff01ull);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double useful = 2.0 * 64 * 32 * ON / 8.0 * iters * (double)blocks * 256 / 32;  // FMAs per lane... per thread
  double instrs = 32.0 * iters * blocks * 256 / 32;  // warp-level FFMA2 issued
  printf("on=%d/8: %.3f ms  useful %.1f TFLOP/s  FFMA2 issue rate %.2f per SMSP-cycle @1.9GHz  %s\n", ON, ms,
         2.0 * 2 * 32 * ON / 8.0 * iters * (double)blocks * 256 / ms / 1e9,
         instrs / (ms * 1e-3) / (148 * 4 * 1.92e9), cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<8>(0xff);
  run<4>(0x55);
  run<2>(0x11);
  run<1>(0x01);
  run<0>(0x00);
}
