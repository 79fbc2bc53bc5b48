// Probe: a dense-kernel inner loop (kernel_dense.cu: 8 output rows per warp as 4
// row pairs, 2 x 7 pixels per lane, 9 taps per input channel) where each (row pair,
// tap) block of 14 FFMA2 runs only if the pair has a nonzero at that tap -- a
// warp-uniform 36-bit mask per channel.  Compares (0) predicated FFMA2 (the block is
// issued with a false predicate), (1) a uniform branch around the block, (2) every
// block (dense).  Masks are random with P(pair active) = p.  Reports executed-block
// fraction, useful (pair-active) TFLOP/s counted as 2 FMAs per active row, and the
// FFMA2-pipe view.  Usage: skip_probe [p_row]
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int S = 7, T = 2, NCH = 96;

template <int MODE>
__global__ void __launch_bounds__(256, 1)
    k(const uint64_t *masks, const float *wts, int iters, float *out, int *active_rows) {
    __shared__ uint64_t sm[NCH];
    __shared__ float4 sw[NCH * 9 * 2];
    __shared__ float win[2048];
    for (int i = threadIdx.x; i < NCH; i += 256) sm[i] = masks[i];
    for (int i = threadIdx.x; i < NCH * 9 * 2; i += 256)
        sw[i] = make_float4(wts[4 * i], wts[4 * i + 1], wts[4 * i + 2], wts[4 * i + 3]);
    for (int i = threadIdx.x; i < 2048; i += 256) win[i] = 0.001f * (i % 97);
    __syncthreads();
    float2 acc[4][T][S];
    for (int p = 0; p < 4; ++p)
        for (int t = 0; t < T; ++t)
            for (int q = 0; q < S; ++q) acc[p][t][q] = make_float2(0.f, 0.f);
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
            float xw[T + 2][S + 2];
#pragma unroll
            for (int r = 0; r < T + 2; ++r)
#pragma unroll
                for (int q = 0; q < S + 2; ++q) xw[r][q] = win[((c & 3) * 5 + r) * 68 + 7 * (lane & 7) + q + (lane >> 3) * 8];
            const uint64_t m = sm[c];
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
                const int ky = tap / 3, kx = tap % 3;
                const float4 w0 = sw[(c * 9 + tap) * 2], w1 = sw[(c * 9 + tap) * 2 + 1];
                const float2 wp[4] = {make_float2(w0.x, w0.y), make_float2(w0.z, w0.w), make_float2(w1.x, w1.y),
                                      make_float2(w1.z, w1.w)};
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const uint32_t bit = uint32_t(m >> (tap * 4 + p)) & 1u;
                    if (MODE == 2 || bit) {
#pragma unroll
                        for (int t = 0; t < T; ++t)
#pragma unroll
                            for (int q = 0; q < S; ++q) {
                                const float xv = xw[t + ky][q + kx];
                                acc[p][t][q] = __ffma2_rn(make_float2(xv, xv), wp[p], acc[p][t][q]);
                            }
                    }
                }
            }
        }
    }
    float s = 0;
    for (int p = 0; p < 4; ++p)
        for (int t = 0; t < T; ++t)
            for (int q = 0; q < S; ++q) s += acc[p][t][q].x + acc[p][t][q].y;
    out[blockIdx.x * 256 + threadIdx.x] = s;
}

int main(int argc, char **argv) {
    const double prow = argc > 1 ? atof(argv[1]) : 0.2;
    std::vector<uint64_t> masks(NCH);
    srand(7);
    long long active_pairs = 0, active_rows = 0;
    for (int c = 0; c < NCH; ++c) {
        uint64_t m = 0;
        for (int i = 0; i < 36; ++i) {
            const bool r0 = rand() < prow * RAND_MAX, r1 = rand() < prow * RAND_MAX;
            if (r0 || r1) { m |= 1ull << i; ++active_pairs; }
            active_rows += r0 + r1;
        }
        masks[c] = m;
    }
    std::vector<float> w(NCH * 9 * 8, 0.5f);
    uint64_t *dm; float *dw, *out; int *dar;
    cudaMalloc(&dm, NCH * 8); cudaMalloc(&dw, w.size() * 4); cudaMalloc(&out, 148 * 256 * 4); cudaMalloc(&dar, 4);
    cudaMemcpy(dm, masks.data(), NCH * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dw, w.data(), w.size() * 4, cudaMemcpyHostToDevice);
    const int iters = 40;
    auto run = [&](auto kern, const char *name) {
        kern<<<148, 256>>>(dm, dw, 1, out, dar);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        kern<<<148, 256>>>(dm, dw, iters, out, dar);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        // per warp per channel: dense = 36 blocks x 14 FFMA2 x 64 FMA
        const double lanes = 148.0 * 256;
        const double useful = 2.0 * (double)active_rows / NCH * 14 * NCH * iters * lanes;  // 2 FLOP per row FMA
        const double dense = 2.0 * 72 * 14 * NCH * iters * lanes;
        printf("p_row=%.2f active pairs %.3f  %-10s %.3f ms  useful %.1f TFLOP/s (%.1f%% of 74.4)  dense-equiv %.1f TFLOP/s  %s\n",
               prow, double(active_pairs) / (36.0 * NCH), name, ms, useful / ms / 1e9, useful / ms / 1e9 / 74.4 * 100,
               dense / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    run(k<0>, "skip-if");
    run(k<2>, "dense");
    return 0;
}
