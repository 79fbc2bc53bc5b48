/*
 * lstm_oracle.c — plain CPU oracle for the sparse multilayer LSTM of
 * SURVEY.md §8(f) NEXT-4 (PAPER.md L422-427 [§RNN]: "iteration space skewing
 * which exposes wavefront parallelism hidden in multilayer-LSTMs"; L510:
 * "4 LSTM layers, 100 elements in the input sequence and 1024 hidden
 * parameters ... 15% as a uniformly distributed density level"; L520: "fuses
 * multiple matrix multiplications into fewer multiplications").
 *
 * TEST INFRASTRUCTURE ONLY (imported by tests/ and scripts' CPU baselines).  It
 * shares no code with the CUDA path.
 *
 * The paper gives no cell equations; reading R3 takes the standard
 * LSTM (the same as torch.nn.LSTM, gate order i, f, g, o):
 *   a = G_l [x ; h_prev] + b_l          (G_l: 4H x (D_l + H) in CSR, the input
 *                                         and recurrent matrices fused, L520)
 *   i = s(a_i), f = s(a_f), g = tanh(a_g), o = s(a_o),  s(v) = 1 / (1 + exp(-v))
 *   c = f * c_prev + i * g,  h = o * tanh(c)
 * with h, c = 0 before t = 0; layer l > 0 consumes layer l-1's h at the same t.
 * Executed sequentially (l outer, t inner), in double precision.
 *
 * Layout: x [T][B][D]; the output h_top [T][B][H] is the last layer's h.
 * CSR of layer l: rows 4H, columns D_l + H (D_0 = D, D_l = H for l > 0),
 * rowptr_all[l*(4H+1) + r] relative to that layer's first nonzero, which is at
 * nnz_off[l] in colidx_all / values_all.  bias_all [L][4H].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double sigm(double v) { return 1.0 / (1.0 + exp(-v)); }

int oracle_lstm_f64(int L, int D, int H, int T, int B, const int32_t *rowptr_all, const int64_t *nnz_off,
                    const int32_t *colidx_all, const float *values_all, const float *bias_all,
                    const float *x, double *h_top) {
    if (L < 1 || D < 1 || H < 1 || T < 1 || B < 1) return -2;
    double *h = calloc((size_t)L * B * H, sizeof(double));  /* h[l][b][k] at the previous step */
    double *c = calloc((size_t)L * B * H, sizeof(double));
    double *z = malloc(sizeof(double) * (size_t)(D > H ? D : H) + sizeof(double) * (size_t)H);
    double *a = malloc(sizeof(double) * 4 * (size_t)H);
    double *below = malloc(sizeof(double) * (size_t)H);
    if (!h || !c || !z || !a || !below) {
        free(h); free(c); free(z); free(a); free(below);
        return -8;
    }
    for (int t = 0; t < T; ++t) {
        for (int b = 0; b < B; ++b) {
            for (int l = 0; l < L; ++l) {
                const int Dl = l == 0 ? D : H;
                /* z = [input ; h_prev] */
                for (int j = 0; j < Dl; ++j)
                    z[j] = l == 0 ? (double)x[((size_t)t * B + b) * D + j] : below[j];
                for (int k = 0; k < H; ++k) z[Dl + k] = h[((size_t)l * B + b) * H + k];
                const int32_t *rp = rowptr_all + (size_t)l * (4 * H + 1);
                const int32_t *ci = colidx_all + nnz_off[l];
                const float *vv = values_all + nnz_off[l];
                for (int r = 0; r < 4 * H; ++r) {
                    double s = 0.0;
                    for (int32_t j = rp[r]; j < rp[r + 1]; ++j) s += (double)vv[j] * z[ci[j]];
                    a[r] = s + (double)bias_all[(size_t)l * 4 * H + r];
                }
                for (int k = 0; k < H; ++k) {
                    const double ig = sigm(a[k]), fg = sigm(a[H + k]);
                    const double gg = tanh(a[2 * H + k]), og = sigm(a[3 * H + k]);
                    double *cp = &c[((size_t)l * B + b) * H + k];
                    *cp = fg * *cp + ig * gg;
                    const double hv = og * tanh(*cp);
                    h[((size_t)l * B + b) * H + k] = hv;
                    below[k] = hv;
                }
            }
            for (int k = 0; k < H; ++k) h_top[((size_t)t * B + b) * H + k] = below[k];
        }
    }
    free(h); free(c); free(z); free(a); free(below);
    return 0;
}
