// Probe: dispatcher with odd window pairs in registers (all taps FFMA2), R = 2, 3, 4
// rows, 8x4 tiles, vs the production-style variant with scalar kx = 1 (gen(4,8,4)).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "probe_odd.inc"
#include "../../paper_2005_04091_b200/csrc/dispatch2_gen.inc"

template <int R, int ODD>
__global__ void __launch_bounds__(256, 1) k(const uint4* stream, int len, int reps, float* out) {
  extern __shared__ uint4 sst[];
  for (int i = threadIdx.x; i < len + 2; i += blockDim.x) sst[i] = stream[i];
  __shared__ __align__(16) uint64_t win[10 * 6 * 32];
  for (int i = threadIdx.x; i < 10 * 6 * 32; i += blockDim.x) win[i] = 0x3f8000003f800000ull + i;
  __syncthreads();
  constexpr int T = 8, S = 4, SH = 2, PAIRS = 3;
  uint64_t acc[R][T][SH];
  for (int r = 0; r < R; ++r) for (int t = 0; t < T; ++t) for (int h = 0; h < SH; ++h) acc[r][t][h] = 0;
  uint64_t xw[T + 2][PAIRS], xo[T + 2][2];
  const uint64_t* wp = win + (threadIdx.x & 31) * 6 * (T + 2);
  for (int i = 0; i < T + 2; ++i) {
    ulonglong2 q = *(const ulonglong2*)(wp + i * 6); xw[i][0] = q.x; xw[i][1] = q.y; xw[i][2] = wp[i * 6 + 2];
    // odd pairs (x1,x2), (x3,x4)
    xo[i][0] = (xw[i][0] >> 32) | (xw[i][1] << 32);
    xo[i][1] = (xw[i][1] >> 32) | (xw[i][2] << 32);
  }
  for (int rep = 0; rep < reps; ++rep) {
    uint32_t sp = (uint32_t)__cvta_generic_to_shared(sst);
    if constexpr (ODD) {
      if constexpr (R == 2) { SPC2_DISPATCHODD_O2T8S4(acc, xw, xo, sp); }
      else if constexpr (R == 3) { SPC2_DISPATCHODD_O3T8S4(acc, xw, xo, sp); }
      else { SPC2_DISPATCHODD_O4T8S4(acc, xw, xo, sp); }
    } else {
      uint32_t wpp = (uint32_t)__cvta_generic_to_shared(win);
      SPC2_DISPATCH_R4T8S4(acc, xw, sp, wpp, 0u, 48u);
    }
  }
  float s = 0; for (int r = 0; r < R; ++r) for (int t = 0; t < T; ++t) for (int h = 0; h < SH; ++h) s += __uint_as_float((uint32_t)acc[r][t][h]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int R, int ODD> void run() {
  const int len = 2000, reps = 200, blocks = 148;
  std::vector<uint4> h(len + 2);
  srand(1);
  for (int i = 0; i < len; ++i) { int c = rand() % (R * 9); h[i] = make_uint4(0x3f800001u, 0x3f800001u, (uint32_t)c, 0); }
  h[len] = make_uint4(0, 0, ODD ? R * 9 : R * 9 + 1, 0); h[len + 1] = h[len];
  uint4* d; cudaMalloc(&d, h.size() * 16); cudaMemcpy(d, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, blocks * 256 * 4);
  size_t smem = h.size() * 16;
  cudaFuncSetAttribute(k<R, ODD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<R, ODD><<<blocks, 256, smem>>>(d, len, 2, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<R, ODD><<<blocks, 256, smem>>>(d, len, reps, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double fl = 2.0 * 32 * (double)len * reps * blocks * 256;
  printf("R=%d odd=%d: %.3f ms  %.1f TFLOP/s (%.0f%%)  %s\n", R, ODD, ms, fl / ms / 1e9, fl / ms / 1e9 / 74.4 * 100,
         cudaGetErrorString(cudaGetLastError()));
}

int main() { run<4, 0>(); run<4, 1>(); run<3, 1>(); run<2, 1>(); }
