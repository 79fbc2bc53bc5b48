/*
 * brute_dense.c — independent pin for the oracle (tests only).
 *
 * Brute-force DENSE direct convolution of the densified filters, written
 * separately from oracle/spconv_oracle.c: explicit zero-padded copy of the
 * input (no bounds tests in the inner loop), seven nested loops in
 * (n, f, oy, ox, c, ky, kx) order — the loop nest of PAPER.md L321-329 —
 * visiting every dense weight including zeros, accumulating with fmaf.
 *
 * Because fmaf(0, x, acc) == acc exactly for finite x and acc != -0, this
 * equals the CSR oracle's FP32-ordered result BITWISE at any sparsity
 * (pin 1).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int brute_dense_conv_f32(int N, int C, int H, int W, int F, int K, int stride, int pad,
                         const float *wdense /* F*C*K*K */, const float *bias /* F or NULL */,
                         const float *x, float *y) {
    const int Hp = H + 2 * pad, Wp = W + 2 * pad;
    const int Ho = (Hp - K) / stride + 1, Wo = (Wp - K) / stride + 1;
    float *xp = (float *)calloc((size_t)N * C * Hp * Wp, sizeof(float));
    if (!xp) return -8;
    for (int n = 0; n < N; ++n)
        for (int c = 0; c < C; ++c)
            for (int i = 0; i < H; ++i)
                memcpy(xp + (((size_t)n * C + c) * Hp + i + pad) * Wp + pad,
                       x + (((size_t)n * C + c) * H + i) * W, sizeof(float) * W);
    for (int n = 0; n < N; ++n)
        for (int f = 0; f < F; ++f)
            for (int oy = 0; oy < Ho; ++oy)
                for (int ox = 0; ox < Wo; ++ox) {
                    float acc = 0.0f;
                    for (int c = 0; c < C; ++c)
                        for (int ky = 0; ky < K; ++ky)
                            for (int kx = 0; kx < K; ++kx) {
                                float w = wdense[(((size_t)f * C + c) * K + ky) * K + kx];
                                float v = xp[(((size_t)n * C + c) * Hp + oy * stride + ky) * Wp +
                                             ox * stride + kx];
                                acc = fmaf(w, v, acc);
                            }
                    y[(((size_t)n * F + f) * Ho + oy) * Wo + ox] = acc + (bias ? bias[f] : 0.0f);
                }
    free(xp);
    return 0;
}
