// kernel_generic.cu — the shape-general CUDA path (any K <= 8, stride, pad).
//
// One thread per output element walks its output channel's CSR row in
// ascending colidx order ("for j in (W.rowptr[n],
// W.rowptr[n+1]) ... out[n][y][x] += coeff*in[...]"), reading the input
// through the read-only cache, and accumulates with FP32 fma in that order
// (reading G7), skipping taps that fall in the zero padding.  Used when the
// tiled kernel does not support the shape, and as a second independent CUDA
// implementation in the parity tests.
#include "spconv_internal.h"

namespace spconv {
namespace {

struct GenericArgs {
    const float *__restrict__ x;
    const int32_t *__restrict__ rowptr;
    const uint32_t *__restrict__ taps;
    const float *__restrict__ values;
    const float *__restrict__ bias;
    int C, H, W, F, stride, pad, Ho, Wo;
};

__device__ __forceinline__ float conv_point(const GenericArgs &a, int n, int f, int oy, int ox) {
    float acc = 0.0f;
    const int j0 = __ldg(a.rowptr + f), j1 = __ldg(a.rowptr + f + 1);
    const float *xn = a.x + (size_t)n * a.C * a.H * a.W;
    const int iy0 = oy * a.stride - a.pad, ix0 = ox * a.stride - a.pad;
    for (int j = j0; j < j1; ++j) {
        const uint32_t t = __ldg(a.taps + j);
        const int c = int(t >> 6), ky = int((t >> 3) & 7u), kx = int(t & 7u);
        const int iy = iy0 + ky, ix = ix0 + kx;
        if (iy < 0 || iy >= a.H || ix < 0 || ix >= a.W) continue; // zero padding
        acc = __fmaf_rn(__ldg(a.values + j), __ldg(xn + ((size_t)c * a.H + iy) * a.W + ix), acc);
    }
    return __fadd_rn(acc, __ldg(a.bias + f));
}

// epi: bit 0 = ReLU, bit 1 = residual add; y = ReLU((acc + bias) + res[i]).
// res may alias y exactly (each element is read, then written, by one thread).
__global__ void __launch_bounds__(256) generic_conv_kernel(GenericArgs a, int64_t total, float *y,
                                                           const float *res, int epi) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ox = int(i % a.Wo);
        int64_t r = i / a.Wo;
        const int oy = int(r % a.Ho);
        r /= a.Ho;
        const int f = int(r % a.F);
        const int n = int(r / a.F);
        float v = conv_point(a, n, f, oy, ox);
        if (epi & 2) v = __fadd_rn(v, res[i]);
        if (epi & 1) v = v > 0.0f ? v : 0.0f;
        y[i] = v;
    }
}

__global__ void __launch_bounds__(256) generic_fused_kernel(GenericArgs a, int64_t total, int Po,
                                                            int Qo, float *__restrict__ y,
                                                            int32_t *__restrict__ argmax) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int px = int(i % Qo);
        int64_t r = i / Qo;
        const int py = int(r % Po);
        r /= Po;
        const int f = int(r % a.F);
        const int n = int(r / a.F);
        float best = 0.0f;
        int bidx = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) { // (0,0), (0,1), (1,0), (1,1): row-major window order
            const int oy = 2 * py + (w >> 1), ox = 2 * px + (w & 1);
            const float v = conv_point(a, n, f, oy, ox);
            const float rv = v > 0.0f ? v : 0.0f; // ReLU, +0 for v <= 0 (reading G11)
            if (w == 0 || rv > best) {            // first max under strict '>' (G10)
                best = rv;
                bidx = oy * a.Wo + ox;
            }
        }
        y[i] = best;
        if (argmax) argmax[i] = bidx;
    }
}

GenericArgs make_args(const Plan &p, const float *x) {
    GenericArgs a;
    a.x = x;
    a.rowptr = p.d_rowptr;
    a.taps = p.d_taps;
    a.values = p.d_values;
    a.bias = p.d_bias;
    a.C = p.C; a.H = p.H; a.W = p.W; a.F = p.F;
    a.stride = p.stride; a.pad = p.pad; a.Ho = p.Ho; a.Wo = p.Wo;
    return a;
}

int grid_for(int64_t total) {
    int64_t b = (total + 255) / 256;
    const int64_t cap = 148 * 16; // grid-stride beyond 16 CTAs per SM
    return int(b < cap ? (b > 0 ? b : 1) : cap);
}

} // namespace

cudaError_t launch_generic_conv(const Plan &p, int N, const float *x, float *y, cudaStream_t s,
                                const float *res, int epi) {
    const int64_t total = (int64_t)N * p.F * p.Ho * p.Wo;
    generic_conv_kernel<<<grid_for(total), 256, 0, s>>>(make_args(p, x), total, y, res, epi);
    return cudaGetLastError();
}

cudaError_t launch_generic_fused(const Plan &p, int N, const float *x, float *y, int32_t *argmax,
                                 cudaStream_t s) {
    const int Po = p.Ho / 2, Qo = p.Wo / 2;
    const int64_t total = (int64_t)N * p.F * Po * Qo;
    generic_fused_kernel<<<grid_for(total), 256, 0, s>>>(make_args(p, x), total, Po, Qo, y, argmax);
    return cudaGetLastError();
}

} // namespace spconv
