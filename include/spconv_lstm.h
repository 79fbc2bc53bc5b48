/*
 * spconv_lstm.h — C-ABI of the sparse multilayer LSTM in libspconv.so
 * (SURVEY.md §8(f) NEXT-4).
 *
 * The operation (arXiv 2005.04091, /root/reference/PAPER.md):
 *   * L422-427 [§RNN]: multilayer LSTMs are parallelised by "iteration space
 *     skewing which exposes wavefront parallelism": cell (l, t) depends on
 *     (l, t-1) and (l-1, t), so all cells on an anti-diagonal w = l + t are
 *     independent.
 *   * L510 [§Evaluation]: "4 LSTM layers, 100 elements in the input sequence
 *     and 1024 hidden parameters ... 15% as a uniformly distributed density".
 *   * L520: the input and recurrent matrix products are fused into fewer
 *     multiplications.
 *   * The cell equations are not given; reading R3 takes the
 *     standard LSTM (identical to torch.nn.LSTM, gate order i, f, g, o):
 *       a = G_l [x ; h_prev] + b_l,  G_l = [W_l | U_l] (4H x (D_l + H), CSR)
 *       i = s(a_i), f = s(a_f), g = tanh(a_g), o = s(a_o), s(v) = 1/(1+e^-v)
 *       c = f*c_prev + i*g,  h = o*tanh(c);  h = c = 0 before t = 0.
 *     Each gate row is a FP32 fma chain in ascending column order.
 *
 * Ownership and errors as spconv.h: the CSR is deep-copied at create (host or
 * device pointers); x / h_top are caller-owned device buffers; every argument
 * is checked before any launch (negative SPCONV_ERR_* codes, spconv.h);
 * forwards are asynchronous on `stream`; T (the sequence length) is a call
 * argument, not a plan constant (the paper's dynamic-RNN point, L415-421).
 */
#ifndef SPCONV_LSTM_H_
#define SPCONV_LSTM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct spconv_lstm_s *spconv_lstm_t;

enum { SPCONV_LSTM_WAVEFRONT = 0, SPCONV_LSTM_SEQUENTIAL = 1 };

/* Layer l's fused gate matrix has 4H rows and D_l + H columns (D_0 = D, D_l = H
 * for l > 0; columns [0, D_l) multiply the layer input, [D_l, D_l + H) the
 * previous hidden state).  rowptr_all: L*(4H+1) int32, each layer's rowptr
 * relative to its first nonzero; nnz_off: L+1 int64, layer l's nonzeros are
 * colidx_all / values_all [nnz_off[l], nnz_off[l+1]); columns strictly
 * ascending per row; bias_all: L*4H floats or NULL (= 0). */
int spconv_lstm_create(spconv_lstm_t *plan, int L, int D, int H, const int32_t *rowptr_all,
                       const int64_t *nnz_off, const int32_t *colidx_all, const float *values_all,
                       const float *bias_all, int device);

/* h_top[T][B][H] = the last layer's hidden states for input x[T][B][D]
 * (device float buffers, not overlapping).  schedule: SPCONV_LSTM_WAVEFRONT
 * (one launch per anti-diagonal, up to L cells in flight) or
 * SPCONV_LSTM_SEQUENTIAL (one launch per cell, l outer, t inner).  The state
 * history lives in a stream-ordered device workspace.  T == 0 or B == 0 is a
 * no-op. */
int spconv_lstm_forward(spconv_lstm_t plan, int T, int B, const float *x, float *h_top, int schedule,
                        void *stream);

/* Kernel launches one forward issues for (T, schedule), or a negative code. */
int spconv_lstm_launches(spconv_lstm_t plan, int T, int schedule);

int spconv_lstm_destroy(spconv_lstm_t plan);

#ifdef __cplusplus
}
#endif
#endif /* SPCONV_LSTM_H_ */
