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
#include <cstdlib>
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
    // staged kernel (H % 8 == 0): entries grouped per (layer, chunk, 8-unit block)
    int32_t *d_off = nullptr; // [L][nzc][4H + 4]
    int2 *d_ent = nullptr;
    int nzc = 0, ent_cap = 0;
    int64_t nnz = 0;
    // A/B knobs, read once at create: SPCONV_LSTM_KERNEL=rowwarp, SPCONV_LSTM_WPC=8|16
    bool force_rowwarp = false;
    int force_wpc = 0;
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

// Batches B >= 32 with B % 4 == 0 (16-byte rows) and H % 8 == 0: the z-staged
// kernel.  CTA = WPC warps = WPC consecutive hidden units of one cell and a tile of
// 64 batch columns; warp w owns unit k0 + w (its four gate rows i, f, g, o), lane =
// batch columns b0 + 2*lane, +1.  Per chunk of ZC rows of the stacked operand
// z = [input ; h_prev], one cp.async stage (double-buffered) brings into shared
// memory (i) the ZC x 64 z tile and (ii) the CTA's nonzeros in that chunk, which
// create() laid out contiguously per (layer, chunk, block of 8 units) as 16-byte
// aligned groups of {col * ZROW, value} entries with their per-row offsets.  So the
// walk touches only shared memory: per nonzero one broadcast LDS.64 (entry), one
// LDS.64 (z), two fma.  Rows' entries stay in ascending column order and chunks
// ascend, so every gate is the same fma chain as in lstm_cells_kernel (bitwise
// identical results).
constexpr int ZC = 128;         // z rows per staged chunk (measured: 32 and 64 slower; per-chunk overhead)
constexpr int ZROW = 64 * 4;    // bytes per staged z row (64 batch columns)
constexpr int LSTM_NSTG = 2;    // cp.async stages in flight (3 measured slower: fewer CTAs per SM)

struct StagedArgs {
    CellArgs a;
    const int2 *ent;    // entries, grouped per (layer, chunk, 8-unit block), groups 16-byte aligned
    const int32_t *off; // [L][nzc][4H + 4]: entry index of row-local q = kb8*32 + g*8 + w; [4H] = end
    int nzc;            // chunks per layer = ceil((max(D, H) + H) / ZC)
    int ent_cap;        // entries per stage buffer (max over CTA blocks and chunks, even)
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}

// One gate row's entries [j, je) of the staged entry buffer, in order (the row's
// fma chain), 4 per round so four LDS chains are in flight; no per-entry predicates
// (ncu: a predicated 4-row interleave was ALU-issue bound at 25 instructions per nonzero).
__device__ __forceinline__ void walk_row(const int2 *es, int j, int je, const unsigned char *zb, float &a0,
                                         float &a1) {
    for (; j + 4 <= je; j += 4) {
        int2 e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) e[u] = es[j + u];
        float2 z[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) z[u] = *reinterpret_cast<const float2 *>(zb + e[u].x);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float v = __int_as_float(e[u].y);
            a0 = __fmaf_rn(v, z[u].x, a0);
            a1 = __fmaf_rn(v, z[u].y, a1);
        }
    }
    for (; j < je; ++j) {
        const int2 e = es[j];
        const float2 z = *reinterpret_cast<const float2 *>(zb + e.x);
        const float v = __int_as_float(e.y);
        a0 = __fmaf_rn(v, z.x, a0);
        a1 = __fmaf_rn(v, z.y, a1);
    }
}

template <int WPC>
__global__ void __launch_bounds__(WPC * 32) lstm_cells_staged_kernel(const StagedArgs sa) {
    const CellArgs &a = sa.a;
    // dynamic smem: [LSTM_NSTG stages][ZC * ZROW z bytes | ent_cap * 8 entry bytes | (4*WPC + 4) offsets]
    extern __shared__ __align__(16) unsigned char dsm[];
    constexpr int NQ = 4 * WPC;                 // gate rows of the CTA
    const uint32_t ent_bytes = uint32_t(sa.ent_cap) * 8u;
    const uint32_t stage_bytes = uint32_t(ZC * ZROW) + ent_bytes + uint32_t(NQ + 4) * 4u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nkb = a.H / WPC;
    const int bt = blockIdx.x % a.nbc;
    const int kb = (blockIdx.x / a.nbc) % nkb;
    const int ci = blockIdx.x / (a.nbc * nkb);
    const int l = a.l0 + ci, t = a.w - l;
    const int k = kb * WPC + warp;
    const int Dl = l == 0 ? a.D : a.H, ncol = Dl + a.H;
    const int nch = (ncol + ZC - 1) / ZC;
    const size_t HB = size_t(a.H) * a.B;
    const float *in = l == 0 ? a.xT + size_t(t) * a.D * a.B
                             : a.hist + (size_t(l - 1) * (a.T + 1) + (t + 1)) * HB;
    const float *rec = a.hist + (size_t(l) * (a.T + 1) + t) * HB;
    const int b0 = bt * 64;
    const uint32_t sm0 = static_cast<uint32_t>(__cvta_generic_to_shared(dsm));
    const int q0 = kb * WPC * 4;                // first row-local index of the CTA (kb8 * 32)
    const int32_t *offl = sa.off + size_t(l) * sa.nzc * (4 * a.H + 4);

    auto stage = [&](int c, int buf) {
        const uint32_t base = sm0 + uint32_t(buf) * stage_bytes;
        for (int e = threadIdx.x; e < ZC * 16; e += WPC * 32) {
            const int r = e >> 4, q = e & 15;
            const int col = c * ZC + r, b = b0 + 4 * q;
            const bool ok = col < ncol && b < a.B;
            const float *src = ok ? (col < Dl ? in + size_t(col) * a.B : rec + size_t(col - Dl) * a.B) + b : a.xT;
            cp_async16(base + uint32_t(r * ZROW + q * 16), src, ok);
        }
        const int32_t *oc = offl + size_t(c) * (4 * a.H + 4);
        const int e0 = __ldg(oc + q0), e1 = __ldg(oc + q0 + NQ); // group-aligned: even, 16-byte
        for (int i = threadIdx.x; 2 * i < e1 - e0; i += WPC * 32)
            cp_async16(base + uint32_t(ZC * ZROW) + uint32_t(i) * 16u, sa.ent + e0 + 2 * i, true);
        for (int i = threadIdx.x; i <= NQ; i += WPC * 32)
            cp_async4(base + uint32_t(ZC * ZROW) + ent_bytes + uint32_t(i) * 4u, oc + q0 + i);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    float acc[4][2] = {};
    const int w8 = warp >> 3, wl = warp & 7;    // 8-unit block within the CTA, unit within it
    // LSTM_NSTG-deep cp.async ring (empty commit groups keep the group count uniform)
#pragma unroll
    for (int s0 = 0; s0 < LSTM_NSTG - 1; ++s0) {
        if (s0 < nch) stage(s0, s0);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int c = 0; c < nch; ++c) {
        const int cn = c + LSTM_NSTG - 1;
        if (cn < nch) stage(cn, cn % LSTM_NSTG);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(LSTM_NSTG - 1) : "memory");
        __syncthreads();
        const unsigned char *sb = dsm + size_t(c % LSTM_NSTG) * stage_bytes;
        const int2 *es = reinterpret_cast<const int2 *>(sb + ZC * ZROW);
        const int32_t *so = reinterpret_cast<const int32_t *>(sb + ZC * ZROW + ent_bytes);
        // generic pointer such that zb + col * ZROW addresses row col - c * ZC of the tile
        const unsigned char *zb = sb + lane * 8 - ptrdiff_t(c) * ZC * ZROW;
        const int eb = so[0];
        const int qb = w8 * 32 + wl;
        walk_row(es, so[qb] - eb, so[qb + 1] - eb, zb, acc[0][0], acc[0][1]);
        walk_row(es, so[qb + 8] - eb, so[qb + 9] - eb, zb, acc[1][0], acc[1][1]);
        walk_row(es, so[qb + 16] - eb, so[qb + 17] - eb, zb, acc[2][0], acc[2][1]);
        walk_row(es, so[qb + 24] - eb, so[qb + 25] - eb, zb, acc[3][0], acc[3][1]);
        __syncthreads(); // buffer c % LSTM_NSTG is refilled by a later iteration's stage()
    }
    float gate[4][2];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const float bb = __ldg(a.bias + size_t(l) * 4 * a.H + g * a.H + k);
        gate[g][0] = __fadd_rn(acc[g][0], bb);
        gate[g][1] = __fadd_rn(acc[g][1], bb);
    }
    float *cp = a.cst + size_t(l) * HB + size_t(k) * a.B;
    float *hp = a.hist + (size_t(l) * (a.T + 1) + (t + 1)) * HB + size_t(k) * a.B;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int b = b0 + 2 * lane + e;
        if (b >= a.B) continue;
        const float ig = sigm(gate[0][e]), fg = sigm(gate[1][e]);
        const float gg = tanhf(gate[2][e]), og = sigm(gate[3][e]);
        const float cc = __fadd_rn(__fmul_rn(fg, cp[b]), __fmul_rn(ig, gg));
        cp[b] = cc;
        hp[b] = __fmul_rn(og, tanhf(cc));
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
    // nonzeros in flight per lane (measured: B=1 4 -> 1.29 ms, 8 -> 1.49; B=8 8 -> 5.47, 4 -> 5.76)
    constexpr int LSTM_SMALL_U = BL == 1 ? 4 : 8;
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
        // LSTM_SMALL_U of the lane's nonzeros per round: their index/value loads, then their z
        // gathers, are all in flight together (ncu: the one-at-a-time loop was bound by
        // the load latency chain, long_scoreboard 28 warps per issue).  Same order per lane.
        for (int j = j0 + nl; j < j1; j += LSTM_SMALL_U * NL) {
            int col[LSTM_SMALL_U];
            float v[LSTM_SMALL_U], z[LSTM_SMALL_U];
#pragma unroll
            for (int u = 0; u < LSTM_SMALL_U; ++u) {
                const int jj = j + u * NL;
                col[u] = jj < j1 ? __ldg(a.colidx + jj) : 0;
                v[u] = jj < j1 ? __ldg(a.values + jj) : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < LSTM_SMALL_U; ++u) {
                const float *zr = col[u] < Dl ? in + size_t(col[u]) * a.B : rec + size_t(col[u] - Dl) * a.B;
                z[u] = okb ? __ldg(zr + bl) : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < LSTM_SMALL_U; ++u)
                if (okb && j + u * NL < j1) acc = __fmaf_rn(v[u], z[u], acc);
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
    cudaFree(p->d_off);
    cudaFree(p->d_ent);
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
    // staged-kernel layout (H % 8 == 0): for each layer l and chunk c of ZC z rows,
    // for each block of 8 hidden units, the 32 gate rows (q = g*8 + w, row = g*H +
    // 8*kb8 + w) each contribute their nonzeros with column in the chunk, as entries
    // {col * ZROW, value bits}; every block's group is padded to an even count so it
    // starts 16-byte aligned.  off[l][c][kb8*32 + q] = entry index of the row's first.
    const int nzc = (std::max(D, H) + H + ZC - 1) / ZC;
    std::vector<int32_t> offs;
    std::vector<int2> ent;
    int ent_cap = 0;
    if (H % 8 == 0) {
        const size_t stride = size_t(4) * H + 4;
        offs.assign(size_t(L) * nzc * stride, 0);
        ent.reserve(static_cast<size_t>(nnz + int64_t(L) * nzc * (H / 8)));
        std::vector<int32_t> cur(size_t(4) * H);
        for (int l = 0; l < L; ++l) {
            const int32_t *r = rp.data() + size_t(l) * (4 * H + 1);
            for (int row = 0; row < 4 * H; ++row) cur[size_t(row)] = r[row];
            for (int c = 0; c < nzc; ++c) {
                int32_t *o = offs.data() + (size_t(l) * nzc + c) * stride;
                for (int kb8 = 0; kb8 < H / 8; ++kb8) {
                    for (int q = 0; q < 32; ++q) {
                        const int row = (q / 8) * H + kb8 * 8 + q % 8;
                        o[kb8 * 32 + q] = int32_t(ent.size());
                        int32_t &j = cur[size_t(row)];
                        for (; j < r[row + 1] && ci[size_t(j)] < (c + 1) * ZC; ++j) {
                            int vb;
                            std::memcpy(&vb, &vv[size_t(j)], 4);
                            ent.push_back(make_int2(ci[size_t(j)] * ZROW, vb));
                        }
                    }
                    // pad to 16 bytes with a zero-valued entry on a column of this chunk: it
                    // joins the block's last row, and fma(0, z, acc) == acc exactly (z finite,
                    // acc never -0 since every chain starts at +0)
                    if (ent.size() & 1) ent.push_back(make_int2(c * ZC * ZROW, 0));
                }
                for (int e = 4 * H; e < 4 * H + 4; ++e) o[e] = int32_t(ent.size());
                // stage capacity: the largest 16-unit (and 8-unit) span of this chunk
                for (int kb8 = 0; kb8 < H / 8; ++kb8) {
                    const int span = (H % 16 == 0 && kb8 % 2 == 0) ? 2 : 1;
                    ent_cap = std::max(ent_cap, o[std::min(kb8 + span, H / 8) * 32] - o[kb8 * 32]);
                }
            }
        }
        if (ent.size() > size_t(INT32_MAX)) return SPCONV_ERR_UNSUPPORTED;
        if (ent.empty()) ent.push_back(make_int2(0, 0));
    }
    spconv_lstm_s *p = new (std::nothrow) spconv_lstm_s;
    if (!p) return SPCONV_ERR_OOM;
    if (const char *e = std::getenv("SPCONV_LSTM_KERNEL")) p->force_rowwarp = std::strcmp(e, "rowwarp") == 0;
    if (const char *e = std::getenv("SPCONV_LSTM_WPC")) p->force_wpc = std::atoi(e);
    p->L = L; p->D = D; p->H = H; p->device = device; p->nnz = nnz; p->nzc = nzc; p->ent_cap = ent_cap + 2;
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
        (st = up(&p->d_bias, bb)) || (!offs.empty() && ((st = up(&p->d_off, offs)) || (st = up(&p->d_ent, ent))))) {
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
    // B >= 32: the z-staged kernel when rows are 16-byte strided (else one warp per row set)
    const bool rowwarp = p->force_rowwarp; // A/B tooling and tests (read at create)
    bool staged = !rowwarp && B >= 32 && B % 4 == 0 && H % 8 == 0 && p->d_off;
    // dynamic shared memory: LSTM_NSTG stages x (z tile + entry buffer + row offsets)
    const size_t zent = size_t(ZC) * ZROW + size_t(p->ent_cap) * 8;
    const size_t smem16 = LSTM_NSTG * (zent + (4 * 16 + 4) * 4), smem8 = LSTM_NSTG * (zent + (4 * 8 + 4) * 4);
    if (staged) {
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device);
        if (smem16 > size_t(optin) ||
            cudaFuncSetAttribute(lstm_cells_staged_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem16)) != cudaSuccess ||
            cudaFuncSetAttribute(lstm_cells_staged_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem8)) != cudaSuccess) {
            cudaGetLastError();
            staged = false; // very dense layers: the one-warp-per-unit kernel
        }
    }
    const int wpc = p->force_wpc; // A/B tooling: force 8 or 16 warps per CTA (read at create)
    StagedArgs sa;
    sa.off = p->d_off; sa.ent = p->d_ent; sa.nzc = p->nzc; sa.ent_cap = p->ent_cap;
    auto launch = [&](int w, int l0, int ncell) {
        a.w = w; a.l0 = l0; a.ncell = ncell;
        if (staged) {
            sa.a = a;
            // 16 warps per CTA (half the z staging per gate row) when that still gives a
            // CTA per SM (paper size, wavefront: 12.5 -> 9.5 ms); else 8 (sequential)
            if (H % 16 == 0 && wpc != 8 && (wpc == 16 || int64_t(ncell) * (H / 16) * a.nbc >= 148))
                lstm_cells_staged_kernel<16><<<ncell * (H / 16) * a.nbc, 512, smem16, s>>>(sa);
            else
                lstm_cells_staged_kernel<8><<<ncell * (H / 8) * a.nbc, 256, smem8, s>>>(sa);
        } else if (B >= 32) {
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
