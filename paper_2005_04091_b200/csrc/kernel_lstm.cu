// kernel_lstm.cu — sparse multilayer LSTM with the wavefront (iteration-space
// skewing) schedule (include/spconv_lstm.h for the
// contract and the PAPER.md passages: L422-427 skewing, L510 sizes and density,
// L520 fused matrix products).
//
// B200 mapping:
//  * State layout: h history hist[l][t+1][k][b] (slot 0 = the zero initial state)
//    and c[l][k][b], batch innermost so that a warp reading one row of the
//    stacked operand z = [input ; h_prev] for 64 batch columns issues two
//    coalesced 128-byte loads.  The input is transposed once to x^T[t][d][b].
//  * One warp per (cell, hidden unit k, 64-wide batch chunk): it evaluates the four
//    gate rows i, f, g, o of unit k of the fused CSR gate matrix [W | U] (each an
//    FP32 fma chain in ascending column order, then + bias) and applies the cell
//    update in registers, so no gate pre-activation ever reaches memory.  The
//    warp's CSR row is fetched 32 nonzeros at a time (one per lane) and broadcast
//    with shuffles.
//  * Wavefront: one launch per anti-diagonal w = l + t covers every cell of the
//    diagonal (up to L) at once — L times the parallelism of the sequential
//    schedule (one launch per cell), which is kept for comparison.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include "spconv.h"
#include "spconv_internal.h"
#include "spconv_lstm.h"

struct spconv_lstm_s {
    int L = 0, D = 0, H = 0, device = 0;
    int32_t *d_rowptr = nullptr; // [L][4H+1], global nonzero offsets
    int32_t *d_colidx = nullptr;
    float *d_values = nullptr;
    float *d_bias = nullptr; // [L][4H]
    int64_t nnz = 0;
};

namespace {

struct CellArgs {
    const int32_t *rowptr;
    const int32_t *colidx;
    const float *values;
    const float *bias;
    const float *xT;  // [T][D][B]
    float *hist;      // [L][T+1][H][B]
    float *cst;       // [L][H][B]
    int L, D, H, T, B, nbc;
    int w, l0, ncell; // diagonal, first layer, number of cells in this launch
};

__device__ __forceinline__ float sigm(float v) { return 1.0f / (1.0f + expf(-v)); }

__global__ void __launch_bounds__(256) lstm_cells_kernel(const CellArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwork = int64_t(a.ncell) * a.H * a.nbc;
    if (gw >= nwork) return;
    const int bc = int(gw % a.nbc);
    const int k = int((gw / a.nbc) % a.H);
    const int ci = int(gw / (int64_t(a.nbc) * a.H));
    const int l = a.l0 + ci, t = a.w - l;
    const int Dl = l == 0 ? a.D : a.H;
    const size_t HB = size_t(a.H) * a.B;
    const float *in = l == 0 ? a.xT + size_t(t) * a.D * a.B
                             : a.hist + (size_t(l - 1) * (a.T + 1) + (t + 1)) * HB;
    const float *rec = a.hist + (size_t(l) * (a.T + 1) + t) * HB;
    const int b0 = bc * 64 + lane, b1 = b0 + 32;
    const bool ok0 = b0 < a.B, ok1 = b1 < a.B;
    const int32_t *rp = a.rowptr + size_t(l) * (4 * a.H + 1);
    float gate[4][2];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const int r = g * a.H + k;
        const int j0 = __ldg(rp + r), j1 = __ldg(rp + r + 1);
        float acc0 = 0.0f, acc1 = 0.0f;
        for (int jb = j0; jb < j1; jb += 32) {
            const int j = jb + lane;
            const int col_l = j < j1 ? __ldg(a.colidx + j) : 0;
            const float val_l = j < j1 ? __ldg(a.values + j) : 0.0f;
            const int cnt = min(32, j1 - jb);
            for (int q = 0; q < cnt; ++q) {
                const int col = __shfl_sync(0xffffffffu, col_l, q);
                const float v = __shfl_sync(0xffffffffu, val_l, q);
                const float *zr = col < Dl ? in + size_t(col) * a.B : rec + size_t(col - Dl) * a.B;
                if (ok0) acc0 = __fmaf_rn(v, __ldg(zr + b0), acc0);
                if (ok1) acc1 = __fmaf_rn(v, __ldg(zr + b1), acc1);
            }
        }
        const float bb = __ldg(a.bias + size_t(l) * 4 * a.H + r);
        gate[g][0] = __fadd_rn(acc0, bb);
        gate[g][1] = __fadd_rn(acc1, bb);
    }
    float *cp = a.cst + size_t(l) * HB + size_t(k) * a.B;
    float *hp = a.hist + (size_t(l) * (a.T + 1) + (t + 1)) * HB + size_t(k) * a.B;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int b = e ? b1 : b0;
        if (!(e ? ok1 : ok0)) continue;
        const float ig = sigm(gate[0][e]), fg = sigm(gate[1][e]);
        const float gg = tanhf(gate[2][e]), og = sigm(gate[3][e]);
        const float c = __fadd_rn(__fmul_rn(fg, cp[b]), __fmul_rn(ig, gg));
        cp[b] = c;
        hp[b] = __fmul_rn(og, tanhf(c));
    }
}

// Small batches (B < 32): lanes split into NL nonzero slices x BL batch columns
// (BL = smallest power of two >= B, NL = 32 / BL).  Lane (nl, bl) accumulates the
// nonzeros j = nl, nl + NL, ... of each gate row for batch column bl; the NL
// partial sums are then added by a shuffle tree.  (At B = 1 the per-row
// mapping above would leave 31 lanes idle.)  The summation order differs from the
// oracle's (tolerance-based parity, reading R3) but is the same for both schedules.
template <int BL>
__global__ void __launch_bounds__(256) lstm_cells_small_kernel(const CellArgs a) {
    constexpr int NL = 32 / BL;
    const int lane = threadIdx.x & 31;
    const int bl = lane % BL, nl = lane / BL;
    const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwork = int64_t(a.ncell) * a.H;
    if (gw >= nwork) return;
    const int k = int(gw % a.H);
    const int ci = int(gw / a.H);
    const int l = a.l0 + ci, t = a.w - l;
    const int Dl = l == 0 ? a.D : a.H;
    const size_t HB = size_t(a.H) * a.B;
    const float *in = l == 0 ? a.xT + size_t(t) * a.D * a.B
                             : a.hist + (size_t(l - 1) * (a.T + 1) + (t + 1)) * HB;
    const float *rec = a.hist + (size_t(l) * (a.T + 1) + t) * HB;
    const bool okb = bl < a.B;
    const int32_t *rp = a.rowptr + size_t(l) * (4 * a.H + 1);
    float gate[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const int r = g * a.H + k;
        const int j0 = __ldg(rp + r), j1 = __ldg(rp + r + 1);
        float acc = 0.0f;
        for (int j = j0 + nl; j < j1; j += NL) {
            const int col = __ldg(a.colidx + j);
            const float v = __ldg(a.values + j);
            const float *zr = col < Dl ? in + size_t(col) * a.B : rec + size_t(col - Dl) * a.B;
            if (okb) acc = __fmaf_rn(v, __ldg(zr + bl), acc);
        }
#pragma unroll
        for (int o = 16; o >= BL; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
        gate[g] = __fadd_rn(acc, __ldg(a.bias + size_t(l) * 4 * a.H + r));
    }
    if (nl != 0 || !okb) return;
    float *cp = a.cst + size_t(l) * HB + size_t(k) * a.B;
    float *hp = a.hist + (size_t(l) * (a.T + 1) + (t + 1)) * HB + size_t(k) * a.B;
    const float ig = sigm(gate[0]), fg = sigm(gate[1]);
    const float gg = tanhf(gate[2]), og = sigm(gate[3]);
    const float c = __fadd_rn(__fmul_rn(fg, cp[bl]), __fmul_rn(ig, gg));
    cp[bl] = c;
    hp[bl] = __fmul_rn(og, tanhf(c));
}

// x[T][B][D] -> xT[T][D][B]
__global__ void transpose_in_kernel(const float *__restrict__ x, float *__restrict__ xT, int T, int B, int D) {
    const int64_t n = int64_t(T) * B * D;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int b = int(i % B);
        const int64_t r = i / B;
        const int d = int(r % D);
        const int t = int(r / D);
        xT[i] = x[(int64_t(t) * B + b) * D + d];
    }
}

// hist[L-1][t+1][k][b] -> h_top[t][b][k]
__global__ void gather_out_kernel(const float *__restrict__ hist, float *__restrict__ out, int L, int T, int B,
                                  int H) {
    const int64_t n = int64_t(T) * B * H;
    const size_t HB = size_t(H) * B;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int k = int(i % H);
        const int64_t r = i / H;
        const int b = int(r % B);
        const int t = int(r / B);
        out[i] = hist[(size_t(L - 1) * (T + 1) + (t + 1)) * HB + size_t(k) * B + b];
    }
}

int grid_for(int64_t n, int per = 256) { return int(std::min<int64_t>((n + per - 1) / per, 148 * 64)); }

template <typename T>
int fetch(const T *src, int64_t n, std::vector<T> &dst) {
    dst.resize(size_t(n));
    if (n == 0) return SPCONV_OK;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, src) != cudaSuccess) {
        cudaGetLastError();
        at.type = cudaMemoryTypeUnregistered;
    }
    if (at.type == cudaMemoryTypeDevice) {
        if (cudaMemcpy(dst.data(), src, sizeof(T) * size_t(n), cudaMemcpyDeviceToHost) != cudaSuccess)
            return SPCONV_ERR_CUDA;
    } else {
        std::memcpy(dst.data(), src, sizeof(T) * size_t(n));
    }
    return SPCONV_OK;
}

void free_lstm(spconv_lstm_s *p) {
    if (!p) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    cudaFree(p->d_rowptr);
    cudaFree(p->d_colidx);
    cudaFree(p->d_values);
    cudaFree(p->d_bias);
    if (prev >= 0) cudaSetDevice(prev);
    delete p;
}

bool is_device_ptr(const void *ptr, int device) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return (at.type == cudaMemoryTypeDevice && at.device == device) || at.type == cudaMemoryTypeManaged;
}

} // namespace

extern "C" {

int spconv_lstm_create(spconv_lstm_t *plan, int L, int D, int H, const int32_t *rowptr_all,
                       const int64_t *nnz_off, const int32_t *colidx_all, const float *values_all,
                       const float *bias_all, int device) {
    if (!plan) return SPCONV_ERR_NULLPTR;
    *plan = nullptr;
    if (!rowptr_all || !nnz_off) return SPCONV_ERR_NULLPTR;
    if (L < 1 || D < 1 || H < 1) return SPCONV_ERR_SHAPE;
    if (int64_t(4) * H + 1 > INT32_MAX / 2 || int64_t(D) + H > INT32_MAX / 2) return SPCONV_ERR_UNSUPPORTED;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
        cudaGetLastError();
        return SPCONV_ERR_CUDA;
    }
    if (device < 0 || device >= ndev) return SPCONV_ERR_DEVICE;
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return SPCONV_ERR_CUDA;
    struct Restore {
        int d;
        ~Restore() { if (d >= 0) cudaSetDevice(d); }
    } restore{prev};

    std::vector<int64_t> off;
    int st;
    if ((st = fetch(nnz_off, L + 1, off))) return st;
    if (off[0] != 0) return SPCONV_ERR_CSR;
    for (int l = 0; l < L; ++l)
        if (off[size_t(l) + 1] < off[size_t(l)]) return SPCONV_ERR_CSR;
    const int64_t nnz = off[size_t(L)];
    if (nnz > INT32_MAX) return SPCONV_ERR_UNSUPPORTED;
    if (nnz > 0 && (!colidx_all || !values_all)) return SPCONV_ERR_NULLPTR;
    std::vector<int32_t> rp, ci;
    std::vector<float> vv, bb;
    if ((st = fetch(rowptr_all, int64_t(L) * (4 * H + 1), rp))) return st;
    if ((st = fetch(colidx_all, nnz, ci))) return st;
    if ((st = fetch(values_all, nnz, vv))) return st;
    if (bias_all) {
        if ((st = fetch(bias_all, int64_t(L) * 4 * H, bb))) return st;
    } else {
        bb.assign(size_t(L) * 4 * H, 0.0f);
    }
    // validate each layer's CSR and rebase rowptr to global nonzero offsets
    for (int l = 0; l < L; ++l) {
        const int cols = (l == 0 ? D : H) + H;
        int32_t *r = rp.data() + size_t(l) * (4 * H + 1);
        if (r[0] != 0 || int64_t(r[4 * H]) != off[size_t(l) + 1] - off[size_t(l)]) return SPCONV_ERR_CSR;
        for (int row = 0; row < 4 * H; ++row) {
            if (r[row + 1] < r[row]) return SPCONV_ERR_CSR;
            for (int32_t j = r[row]; j < r[row + 1]; ++j) {
                const int64_t g = off[size_t(l)] + j;
                if (ci[size_t(g)] < 0 || ci[size_t(g)] >= cols) return SPCONV_ERR_CSR;
                if (j > r[row] && ci[size_t(g)] <= ci[size_t(g) - 1]) return SPCONV_ERR_CSR;
                if (!std::isfinite(vv[size_t(g)])) return SPCONV_ERR_CSR;
            }
        }
        for (int row = 0; row <= 4 * H; ++row) r[row] += int32_t(off[size_t(l)]);
    }
    for (float b : bb)
        if (!std::isfinite(b)) return SPCONV_ERR_CSR;
    spconv_lstm_s *p = new (std::nothrow) spconv_lstm_s;
    if (!p) return SPCONV_ERR_OOM;
    p->L = L; p->D = D; p->H = H; p->device = device; p->nnz = nnz;
    auto up = [&](auto **dst, const auto &src) -> int {
        const size_t bytes = sizeof(src[0]) * std::max<size_t>(src.size(), 1);
        if (cudaMalloc(reinterpret_cast<void **>(dst), bytes) != cudaSuccess) {
            cudaGetLastError();
            return SPCONV_ERR_OOM;
        }
        if (!src.empty() && cudaMemcpy(*dst, src.data(), sizeof(src[0]) * src.size(), cudaMemcpyHostToDevice) !=
                                cudaSuccess)
            return SPCONV_ERR_CUDA;
        return SPCONV_OK;
    };
    if ((st = up(&p->d_rowptr, rp)) || (st = up(&p->d_colidx, ci)) || (st = up(&p->d_values, vv)) ||
        (st = up(&p->d_bias, bb))) {
        free_lstm(p);
        return st;
    }
    *plan = p;
    return SPCONV_OK;
}

int spconv_lstm_launches(spconv_lstm_t plan, int T, int schedule) {
    if (!plan) return SPCONV_ERR_NULLPTR;
    if (T < 0) return SPCONV_ERR_SHAPE;
    if (T == 0) return 0;
    const int cells = schedule == SPCONV_LSTM_SEQUENTIAL ? plan->L * T : plan->L + T - 1;
    return cells + 2; // + input transpose, output gather
}

int spconv_lstm_forward(spconv_lstm_t plan, int T, int B, const float *x, float *h_top, int schedule,
                        void *stream) {
    if (!plan) return SPCONV_ERR_NULLPTR;
    spconv_lstm_s *p = plan;
    if (T < 0 || B < 0) return SPCONV_ERR_SHAPE;
    if (schedule != SPCONV_LSTM_WAVEFRONT && schedule != SPCONV_LSTM_SEQUENTIAL) return SPCONV_ERR_UNSUPPORTED;
    if (T == 0 || B == 0) return SPCONV_OK;
    if (!x || !h_top) return SPCONV_ERR_NULLPTR;
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(h_top)) & 3) return SPCONV_ERR_ALIGN;
    const size_t xb = size_t(T) * B * p->D * 4, yb = size_t(T) * B * p->H * 4;
    const char *x0 = reinterpret_cast<const char *>(x), *y0 = reinterpret_cast<const char *>(h_top);
    if (x0 < y0 + yb && y0 < x0 + xb) return SPCONV_ERR_ALIAS;
    if (!is_device_ptr(x, p->device) || !is_device_ptr(h_top, p->device)) return SPCONV_ERR_DEVICE;
    int prev = -1;
    cudaGetDevice(&prev);
    if (cudaSetDevice(p->device) != cudaSuccess) return SPCONV_ERR_CUDA;
    struct Restore {
        int d;
        ~Restore() { if (d >= 0) cudaSetDevice(d); }
    } restore{prev};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int L = p->L, D = p->D, H = p->H;
    const size_t HB = size_t(H) * B;
    const size_t xT_n = size_t(T) * D * B, hist_n = size_t(L) * (T + 1) * HB, c_n = size_t(L) * HB;
    float *ws = nullptr;
    spconv::keep_pool_cached();
    if (cudaMallocAsync(reinterpret_cast<void **>(&ws), (xT_n + hist_n + c_n) * 4, s) != cudaSuccess) {
        cudaGetLastError();
        return SPCONV_ERR_OOM;
    }
    float *xT = ws, *hist = ws + xT_n, *cst = hist + hist_n;
    cudaError_t e = cudaSuccess;
    // zero initial states: slot 0 of every layer's history, and c
    for (int l = 0; l < L && e == cudaSuccess; ++l)
        e = cudaMemsetAsync(hist + size_t(l) * (T + 1) * HB, 0, HB * 4, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(cst, 0, c_n * 4, s);
    if (e == cudaSuccess) {
        transpose_in_kernel<<<grid_for(int64_t(xT_n)), 256, 0, s>>>(x, xT, T, B, D);
        e = cudaGetLastError();
    }
    CellArgs a;
    a.rowptr = p->d_rowptr; a.colidx = p->d_colidx; a.values = p->d_values; a.bias = p->d_bias;
    a.xT = xT; a.hist = hist; a.cst = cst;
    a.L = L; a.D = D; a.H = H; a.T = T; a.B = B; a.nbc = (B + 63) / 64;
    auto launch = [&](int w, int l0, int ncell) {
        a.w = w; a.l0 = l0; a.ncell = ncell;
        if (B >= 32) {
            const int64_t threads = int64_t(ncell) * H * a.nbc * 32;
            lstm_cells_kernel<<<int((threads + 255) / 256), 256, 0, s>>>(a);
        } else {
            const int64_t threads = int64_t(ncell) * H * 32;
            const int blocks = int((threads + 255) / 256);
            if (B == 1) lstm_cells_small_kernel<1><<<blocks, 256, 0, s>>>(a);
            else if (B == 2) lstm_cells_small_kernel<2><<<blocks, 256, 0, s>>>(a);
            else if (B <= 4) lstm_cells_small_kernel<4><<<blocks, 256, 0, s>>>(a);
            else if (B <= 8) lstm_cells_small_kernel<8><<<blocks, 256, 0, s>>>(a);
            else if (B <= 16) lstm_cells_small_kernel<16><<<blocks, 256, 0, s>>>(a);
            else lstm_cells_small_kernel<32><<<blocks, 256, 0, s>>>(a);
        }
        return cudaGetLastError();
    };
    if (schedule == SPCONV_LSTM_WAVEFRONT) {
        // skewed iteration space: diagonal w holds cells (l, w - l)
        for (int w = 0; w < L + T - 1 && e == cudaSuccess; ++w) {
            const int l0 = std::max(0, w - T + 1), l1 = std::min(L - 1, w);
            e = launch(w, l0, l1 - l0 + 1);
        }
    } else {
        for (int l = 0; l < L && e == cudaSuccess; ++l)
            for (int t = 0; t < T && e == cudaSuccess; ++t) e = launch(l + t, l, 1);
    }
    if (e == cudaSuccess) {
        gather_out_kernel<<<grid_for(int64_t(T) * B * H), 256, 0, s>>>(hist, h_top, L, T, B, H);
        e = cudaGetLastError();
    }
    cudaError_t e2 = cudaFreeAsync(ws, s);
    if (e == cudaSuccess) e = e2;
    return e == cudaSuccess ? SPCONV_OK : SPCONV_ERR_CUDA;
}

int spconv_lstm_destroy(spconv_lstm_t plan) {
    free_lstm(plan);
    return SPCONV_OK;
}

} // extern "C"
