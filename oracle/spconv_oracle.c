/*
 * spconv_oracle.c — plain, slow, obviously-correct CPU oracle for the CSR
 * sparse direct convolution of arXiv 2005.04091.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header or table with the CUDA path
 * (paper_2005_04091_b200/csrc) and includes nothing from it.
 *
 * What it computes:
 *
 *   CSR construction (¶"Sparse Convolution with CSR"): the
 *   (F, C, K, K) weight tensor is flattened to (F, C*K*K) and its rows are
 *   compressed; colidx = (c*K + ky)*K + kx (reading G1).
 *
 *   Convolution (DSL listing: conv(n,fout,y,x) +=
 *   weights(fout,fin,k0,k1) * input(n,fin,y+k0,x+k1) — cross-correlation,
 *   no kernel flip; readings G3-G6 add explicit stride s and zero pad p):
 *
 *     acc(n,f,oy,ox) = sum_{j=rowptr[f]}^{rowptr[f+1]-1}
 *                        values[j] * X(n, c_j, oy*s + ky_j - p, ox*s + kx_j - p)
 *     X(...) = input if inside [0,H)x[0,W) else 0 (zero padding, reading G6)
 *     conv   = acc + bias[f]                       (bias after the sum, G8)
 *
 *   This is the CSR loop of PAPER.md L393-401 ("for each output channel n,
 *   for j in rowptr[n]..rowptr[n+1]: out[n][y][x] += coeff*in[...]"), with
 *   the garbled index of L399 read as explicit 2-D padded indexing (G2).
 *
 *   Fused block ("Conv-Relu-Maxpool"): r = ReLU(conv) with
 *   ReLU(v) = v > 0 ? v : +0 (G11); pooled = max over the 2x2 / stride 2
 *   window (floor, G9); argmax = first (dy,dx) in row-major order attaining
 *   the max under strict '>' (G10), flat index (2py+dy)*Wo + (2px+dx).
 *
 * Two arithmetic modes:
 *   f32 "ordered": acc starts at +0.0f, for j ascending acc = fmaf(v, X, acc)
 *     (one rounding per step, RNE), out-of-bounds taps skipped; then one FP32
 *     add of the bias.  This is reading G7 — the parity contract.
 *   f64: the same loops in double with fma(), result returned in double.
 *
 * Threading: plain pthreads over disjoint (n, f) planes; every output is
 * computed by exactly one thread with the same sequential loop, so results
 * are independent of the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_ERR_SHAPE -2
#define ORACLE_ERR_CSR -3

/* ------------------------------------------------------------------ */
/* CSR validation                   */
/* ------------------------------------------------------------------ */
int oracle_check_csr(int F, int C, int K, const int32_t *rowptr,
                     const int32_t *colidx, const float *values, int64_t nnz) {
    if (F < 1 || C < 1 || K < 1) return ORACLE_ERR_SHAPE;
    if (rowptr[0] != 0) return ORACLE_ERR_CSR;
    if ((int64_t)rowptr[F] != nnz) return ORACLE_ERR_CSR;
    const int64_t ncol = (int64_t)C * K * K;
    for (int f = 0; f < F; ++f) {
        if (rowptr[f + 1] < rowptr[f]) return ORACLE_ERR_CSR;
        for (int32_t j = rowptr[f]; j < rowptr[f + 1]; ++j) {
            if (colidx[j] < 0 || (int64_t)colidx[j] >= ncol) return ORACLE_ERR_CSR;
            if (j > rowptr[f] && colidx[j] <= colidx[j - 1]) return ORACLE_ERR_CSR;
            if (!isfinite(values[j])) return ORACLE_ERR_CSR;
        }
    }
    return ORACLE_OK;
}

/* Decode colidx -> (c, ky, kx): c = col / K^2, ky = (col / K) mod K, kx = col mod K. */
void oracle_decode(int K, int64_t nnz, const int32_t *colidx, int32_t *c,
                   int32_t *ky, int32_t *kx) {
    for (int64_t j = 0; j < nnz; ++j) {
        int32_t col = colidx[j];
        c[j] = col / (K * K);
        ky[j] = (col / K) % K;
        kx[j] = col % K;
    }
}

/* ------------------------------------------------------------------ */
/* One output value, straight from the definition.                     */
/* ------------------------------------------------------------------ */
typedef struct {
    int N, C, H, W, F, K, stride, pad, Ho, Wo;
    const int32_t *rowptr, *colidx;
    const float *values, *bias, *x;
} layer_t;

static float conv_one_f32(const layer_t *L, int n, int f, int oy, int ox) {
    float acc = 0.0f;
    for (int32_t j = L->rowptr[f]; j < L->rowptr[f + 1]; ++j) {
        int32_t col = L->colidx[j];
        int c = col / (L->K * L->K);
        int ky = (col / L->K) % L->K;
        int kx = col % L->K;
        int iy = oy * L->stride + ky - L->pad;
        int ix = ox * L->stride + kx - L->pad;
        if (iy < 0 || iy >= L->H || ix < 0 || ix >= L->W) continue; /* zero padding */
        float xv = L->x[(((int64_t)n * L->C + c) * L->H + iy) * L->W + ix];
        acc = fmaf(L->values[j], xv, acc);
    }
    float b = L->bias ? L->bias[f] : 0.0f;
    return acc + b;
}

static double conv_one_f64(const layer_t *L, int n, int f, int oy, int ox) {
    double acc = 0.0;
    for (int32_t j = L->rowptr[f]; j < L->rowptr[f + 1]; ++j) {
        int32_t col = L->colidx[j];
        int c = col / (L->K * L->K);
        int ky = (col / L->K) % L->K;
        int kx = col % L->K;
        int iy = oy * L->stride + ky - L->pad;
        int ix = ox * L->stride + kx - L->pad;
        if (iy < 0 || iy >= L->H || ix < 0 || ix >= L->W) continue;
        double xv = L->x[(((int64_t)n * L->C + c) * L->H + iy) * L->W + ix];
        acc = fma((double)L->values[j], xv, acc);
    }
    double b = L->bias ? (double)L->bias[f] : 0.0;
    return acc + b;
}

static float relu_f32(float v) { return v > 0.0f ? v : 0.0f; }

/* ------------------------------------------------------------------ */
/* Plane-parallel driver                                                */
/* ------------------------------------------------------------------ */
enum { MODE_F32 = 0, MODE_F64 = 1, MODE_FUSED = 2 };

typedef struct {
    const layer_t *L;
    int mode;
    void *y;            /* float* or double* */
    int32_t *argmax;    /* fused only, may be NULL */
    int64_t begin, end; /* plane range [begin, end) over n*F */
} job_t;

static void run_planes(const job_t *J) {
    const layer_t *L = J->L;
    for (int64_t p = J->begin; p < J->end; ++p) {
        int n = (int)(p / L->F), f = (int)(p % L->F);
        if (J->mode == MODE_F32) {
            float *y = (float *)J->y + p * (int64_t)L->Ho * L->Wo;
            for (int oy = 0; oy < L->Ho; ++oy)
                for (int ox = 0; ox < L->Wo; ++ox)
                    y[oy * L->Wo + ox] = conv_one_f32(L, n, f, oy, ox);
        } else if (J->mode == MODE_F64) {
            double *y = (double *)J->y + p * (int64_t)L->Ho * L->Wo;
            for (int oy = 0; oy < L->Ho; ++oy)
                for (int ox = 0; ox < L->Wo; ++ox)
                    y[oy * L->Wo + ox] = conv_one_f64(L, n, f, oy, ox);
        } else {
            const int Po = L->Ho / 2, Qo = L->Wo / 2; /* floor: G9 */
            float *y = (float *)J->y + p * (int64_t)Po * Qo;
            int32_t *am = J->argmax ? J->argmax + p * (int64_t)Po * Qo : NULL;
            for (int py = 0; py < Po; ++py)
                for (int px = 0; px < Qo; ++px) {
                    float best = 0.0f;
                    int32_t bidx = 0;
                    for (int w = 0; w < 4; ++w) { /* (0,0),(0,1),(1,0),(1,1) */
                        int oy = 2 * py + w / 2, ox = 2 * px + w % 2;
                        float r = relu_f32(conv_one_f32(L, n, f, oy, ox));
                        if (w == 0 || r > best) {
                            best = r;
                            bidx = oy * L->Wo + ox;
                        }
                    }
                    y[py * Qo + px] = best;
                    if (am) am[py * Qo + px] = bidx;
                }
        }
    }
}

static void *thread_main(void *arg) {
    run_planes((const job_t *)arg);
    return NULL;
}

static int run_all(const layer_t *L, int mode, void *y, int32_t *argmax, int nthreads) {
    int64_t planes = (int64_t)L->N * L->F;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > planes) nthreads = (int)(planes > 0 ? planes : 1);
    if (nthreads == 1) {
        job_t J = {L, mode, y, argmax, 0, planes};
        run_planes(&J);
        return ORACLE_OK;
    }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    job_t *jobs = (job_t *)malloc(sizeof(job_t) * nthreads);
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].L = L;
        jobs[t].mode = mode;
        jobs[t].y = y;
        jobs[t].argmax = argmax;
        jobs[t].begin = planes * t / nthreads;
        jobs[t].end = planes * (t + 1) / nthreads;
        pthread_create(&th[t], NULL, thread_main, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return ORACLE_OK;
}

static int make_layer(layer_t *L, int N, int C, int H, int W, int F, int K, int stride,
                      int pad, const int32_t *rowptr, const int32_t *colidx,
                      const float *values, const float *bias, const float *x) {
    if (N < 0 || C < 1 || H < 1 || W < 1 || F < 1 || K < 1 || stride < 1 || pad < 0)
        return ORACLE_ERR_SHAPE;
    L->N = N; L->C = C; L->H = H; L->W = W; L->F = F; L->K = K;
    L->stride = stride; L->pad = pad;
    L->Ho = (H + 2 * pad - K) / stride + 1;
    L->Wo = (W + 2 * pad - K) / stride + 1;
    if (H + 2 * pad < K || W + 2 * pad < K || L->Ho < 1 || L->Wo < 1) return ORACLE_ERR_SHAPE;
    L->rowptr = rowptr; L->colidx = colidx; L->values = values;
    L->bias = bias; L->x = x;
    return ORACLE_OK;
}

/* y[N][F][Ho][Wo] in the FP32-ordered mode. */
int oracle_conv_f32(int N, int C, int H, int W, int F, int K, int stride, int pad,
                    const int32_t *rowptr, const int32_t *colidx, const float *values,
                    const float *bias, const float *x, float *y, int nthreads) {
    layer_t L;
    int s = make_layer(&L, N, C, H, W, F, K, stride, pad, rowptr, colidx, values, bias, x);
    if (s) return s;
    return run_all(&L, MODE_F32, y, NULL, nthreads);
}

/* y[N][F][Ho][Wo] in double precision (accuracy reference). */
int oracle_conv_f64(int N, int C, int H, int W, int F, int K, int stride, int pad,
                    const int32_t *rowptr, const int32_t *colidx, const float *values,
                    const float *bias, const float *x, double *y, int nthreads) {
    layer_t L;
    int s = make_layer(&L, N, C, H, W, F, K, stride, pad, rowptr, colidx, values, bias, x);
    if (s) return s;
    return run_all(&L, MODE_F64, y, NULL, nthreads);
}

/* pooled[N][F][Ho/2][Wo/2] (+ argmax) of ReLU(conv) in the FP32-ordered mode. */
int oracle_fused_f32(int N, int C, int H, int W, int F, int K, int stride, int pad,
                     const int32_t *rowptr, const int32_t *colidx, const float *values,
                     const float *bias, const float *x, float *pooled, int32_t *argmax,
                     int nthreads) {
    layer_t L;
    int s = make_layer(&L, N, C, H, W, F, K, stride, pad, rowptr, colidx, values, bias, x);
    if (s) return s;
    return run_all(&L, MODE_FUSED, pooled, argmax, nthreads);
}

/* Selected outputs, one by one: pts = npts x (n, f, oy, ox). */
int oracle_conv_points_f32(int N, int C, int H, int W, int F, int K, int stride, int pad,
                           const int32_t *rowptr, const int32_t *colidx,
                           const float *values, const float *bias, const float *x,
                           int64_t npts, const int64_t *pts, float *out) {
    layer_t L;
    int s = make_layer(&L, N, C, H, W, F, K, stride, pad, rowptr, colidx, values, bias, x);
    if (s) return s;
    for (int64_t i = 0; i < npts; ++i) {
        const int64_t *p = pts + 4 * i;
        out[i] = conv_one_f32(&L, (int)p[0], (int)p[1], (int)p[2], (int)p[3]);
    }
    return ORACLE_OK;
}

int oracle_conv_points_f64(int N, int C, int H, int W, int F, int K, int stride, int pad,
                           const int32_t *rowptr, const int32_t *colidx,
                           const float *values, const float *bias, const float *x,
                           int64_t npts, const int64_t *pts, double *out) {
    layer_t L;
    int s = make_layer(&L, N, C, H, W, F, K, stride, pad, rowptr, colidx, values, bias, x);
    if (s) return s;
    for (int64_t i = 0; i < npts; ++i) {
        const int64_t *p = pts + 4 * i;
        out[i] = conv_one_f64(&L, (int)p[0], (int)p[1], (int)p[2], (int)p[3]);
    }
    return ORACLE_OK;
}

/* Selected pooled outputs: pts = npts x (n, f, py, px) -> value, argmax. */
int oracle_fused_points_f32(int N, int C, int H, int W, int F, int K, int stride, int pad,
                            const int32_t *rowptr, const int32_t *colidx,
                            const float *values, const float *bias, const float *x,
                            int64_t npts, const int64_t *pts, float *out, int32_t *argmax) {
    layer_t L;
    int s = make_layer(&L, N, C, H, W, F, K, stride, pad, rowptr, colidx, values, bias, x);
    if (s) return s;
    for (int64_t i = 0; i < npts; ++i) {
        const int64_t *p = pts + 4 * i;
        float best = 0.0f;
        int32_t bidx = 0;
        for (int w = 0; w < 4; ++w) {
            int oy = 2 * (int)p[2] + w / 2, ox = 2 * (int)p[3] + w % 2;
            float r = relu_f32(conv_one_f32(&L, (int)p[0], (int)p[1], oy, ox));
            if (w == 0 || r > best) {
                best = r;
                bidx = oy * L.Wo + ox;
            }
        }
        out[i] = best;
        argmax[i] = bidx;
    }
    return ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* Block epilogue for chained layers (DESIGN.md */
/* reading R1): y = ReLU((conv + bias) + residual), in that order, one */
/* FP32 add each; ReLU(v) = v > 0 ? v : +0 (G11).  Applied in place to */
/* the output of oracle_conv_f32.  flags: bit 0 ReLU, bit 1 residual.  */
/* ------------------------------------------------------------------ */
void oracle_epilogue_f32(float *y, const float *residual, int64_t n, int flags) {
    for (int64_t i = 0; i < n; ++i) {
        float v = y[i];
        if (flags & 2) v = v + residual[i];
        if (flags & 1) v = v > 0.0f ? v : 0.0f;
        y[i] = v;
    }
}

/* ------------------------------------------------------------------ */
/* Bilinear resize (SURVEY.md §8(f) NEXT-2 "Resize-Conv-Relu-Maxpool",  */
/* PAPER.md L503; the paper does not define the resize: DESIGN.md      */
/* reading R2 = bilinear, half-pixel centres (align_corners = False),  */
/* source coordinate clamped below at 0, neighbours clamped to the     */
/* image).  Plain FP32 arithmetic in this exact order, no contraction: */
/*   s  = (o + 0.5) * (in / out) - 0.5, s = max(s, 0)                  */
/*   i0 = floor(s), i1 = min(i0 + 1, in - 1), l = s - i0, h = 1 - l    */
/*   v  = hy * (hx*v00 + lx*v01) + ly * (hx*v10 + lx*v11)              */
/* ------------------------------------------------------------------ */
static void resize_coord(int o, int in, int out, int *i0, int *i1, float *l, float *h) {
    float scale = (float)in / (float)out;
    float s = ((float)o + 0.5f) * scale - 0.5f;
    if (s < 0.0f) s = 0.0f;
    int a = (int)s;
    if (a > in - 1) a = in - 1;
    *i0 = a;
    *i1 = a + 1 < in ? a + 1 : in - 1;
    *l = s - (float)a;
    *h = 1.0f - *l;
}

void oracle_resize_bilinear_f32(int N, int C, int Hin, int Win, int Hout, int Wout, const float *x,
                                float *y) {
    for (int64_t nc = 0; nc < (int64_t)N * C; ++nc) {
        const float *src = x + nc * Hin * Win;
        float *dst = y + nc * Hout * Wout;
        for (int oy = 0; oy < Hout; ++oy) {
            int y0, y1;
            float ly, hy;
            resize_coord(oy, Hin, Hout, &y0, &y1, &ly, &hy);
            for (int ox = 0; ox < Wout; ++ox) {
                int x0, x1;
                float lx, hx;
                resize_coord(ox, Win, Wout, &x0, &x1, &lx, &hx);
                float t0 = hx * src[y0 * Win + x0];
                float t1 = lx * src[y0 * Win + x1];
                float a = t0 + t1;
                float t2 = hx * src[y1 * Win + x0];
                float t3 = lx * src[y1 * Win + x1];
                float b = t2 + t3;
                float u = hy * a;
                float w = ly * b;
                dst[oy * Wout + ox] = u + w;
            }
        }
    }
}
