// kernel_resize.cu — bilinear resize prologue of the Resize-Conv-Relu-Maxpool block
// ("the same benchmark as the previous one but
// preceded by an image resizing step for preprocessing").  The paper does not define
// the resize; reading R2 fixes it as bilinear with half-pixel centres
// (align_corners = False), the source coordinate clamped below at 0 and neighbours
// clamped to the image, evaluated in plain FP32 in exactly this order (no fma
// contraction, so the result is bit-identical to the oracle):
//   s = (o + 0.5) * (in / out) - 0.5, s = max(s, 0); i0 = floor(s); i1 = min(i0+1, in-1)
//   l = s - i0, h = 1 - l;  v = hy*(hx*v00 + lx*v01) + ly*(hx*v10 + lx*v11)
#include "spconv_internal.h"

namespace spconv {
namespace {

__device__ __forceinline__ void coord(int o, int in, float scale, int &i0, int &i1, float &l, float &h) {
    float s = __fsub_rn(__fmul_rn(__fadd_rn(float(o), 0.5f), scale), 0.5f);
    if (s < 0.0f) s = 0.0f;
    int a = int(s);
    if (a > in - 1) a = in - 1;
    i0 = a;
    i1 = a + 1 < in ? a + 1 : in - 1;
    l = __fsub_rn(s, float(a));
    h = __fsub_rn(1.0f, l);
}

__global__ void __launch_bounds__(256) resize_bilinear_kernel(const float *__restrict__ x, float *__restrict__ y,
                                                              int64_t planes, int Hin, int Win, int Hout,
                                                              int Wout) {
    const float sy = __fdiv_rn(float(Hin), float(Hout)), sx = __fdiv_rn(float(Win), float(Wout));
    const int64_t total = planes * Hout * Wout;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ox = int(i % Wout);
        const int64_t r = i / Wout;
        const int oy = int(r % Hout);
        const int64_t pl = r / Hout;
        int y0, y1, x0, x1;
        float ly, hy, lx, hx;
        coord(oy, Hin, sy, y0, y1, ly, hy);
        coord(ox, Win, sx, x0, x1, lx, hx);
        const float *src = x + pl * Hin * Win;
        const float t0 = __fmul_rn(hx, __ldg(src + y0 * Win + x0));
        const float t1 = __fmul_rn(lx, __ldg(src + y0 * Win + x1));
        const float t2 = __fmul_rn(hx, __ldg(src + y1 * Win + x0));
        const float t3 = __fmul_rn(lx, __ldg(src + y1 * Win + x1));
        const float a = __fadd_rn(t0, t1), b = __fadd_rn(t2, t3);
        y[i] = __fadd_rn(__fmul_rn(hy, a), __fmul_rn(ly, b));
    }
}

} // namespace

cudaError_t launch_resize(const float *x, float *y, int64_t planes, int Hin, int Win, int Hout, int Wout,
                          cudaStream_t s) {
    const int64_t total = planes * Hout * Wout;
    const int blocks = int(std::min<int64_t>((total + 255) / 256, 148 * 32));
    resize_bilinear_kernel<<<blocks, 256, 0, s>>>(x, y, planes, Hin, Win, Hout, Wout);
    return cudaGetLastError();
}

} // namespace spconv
