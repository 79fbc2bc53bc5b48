// kernel_dense.cu -- dense FP32 direct convolution (K = 3, stride 1, pad 1) on sm_100a:
// the "dense convolution implementation" the paper's break-even density is measured
// against (¶Evaluation: "a dense convolution implementation is more
// profitable than the sparse counterpart" above 43.5% density).
//
// It computes the same operation as the sparse kernels from the DENSIFIED filters
// (CSR is a lossless compression of the (F, C*K*K) matrix): per output,
// FP32 fma over every (c, ky, kx) in ascending order, then one FP32 add of the bias.
// A zero filter tap is an exact no-op (fma(0, x, acc) == acc for finite x, and acc is
// never -0 when it starts at +0), so the result is BITWISE the FP32-ordered oracle's
// for any sparsity pattern -- the sparse and dense paths are interchangeable, which is
// what lets AUTO route dense-enough layers here.
//
// Mapping (static code, no per-nonzero dispatch):
//  * CTA = 8 warps (2 per SM sub-partition, up to 255 registers).  Warp w owns output channels
//    [fset*64 + 8w, +8); lane (lx, ly) owns a T x S = 2 x S output tile (S = 7 or 8,
//    LR = lanes per staged row, LY = lane rows), so a thread holds 8 x 2 x S
//    accumulators.
//  * Accumulators are pairs of OUTPUT CHANNELS at one pixel: one packed
//    fma.rn.f32x2 (FFMA2) updates channels (2p, 2p+1) with the weight pair
//    (w[2p], w[2p+1]) and the input value broadcast -- so any tap offset, including
//    the odd kx = 1 shift, is one FFMA2 per pixel and channel pair (no pixel-pair
//    alignment constraint).  Per input channel: 9 taps x 4 pairs x 2S pixels FFMA2.
//  * Staging: per stage cc input channels of the unit's rows (+ halo) by one 4-D TMA
//    box (out-of-bounds zero fill = the padding) and the stage's weight slab
//    [warp][c][tap][8] by one bulk copy, both on the stage's mbarrier; an mbarrier ring
//    of nstage stages; the last warp to release a stage refills it.  Window words are read with LDS.32
//    at a pitch chosen for conflict-free banks; the 8 weights of a tap by two
//    warp-uniform LDS.128 (broadcast).
//  * Persistent CTAs over (pixel block, 64-channel set) units.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "async_copy.cuh"
#include "spconv_internal.h"

namespace spconv {
namespace {
using namespace dev;

constexpr int DW = 8;        // consumer warps per CTA
constexpr int DR = 8;        // output channels per warp
constexpr int DT = 2;        // output rows per lane tile
constexpr int DMAXSTAGE = 8;

struct DenseArgs {
    const float *x, *bias, *wslab;
    const float *res; // residual added before the optional ReLU (epi & 2); may alias y
    float *y;
    int32_t *argmax;  // fused: first-max flat index per pooled output, or null
    int epi;          // conv-only epilogue: bit 0 ReLU, bit 1 residual (reading R1)
    int Po, Qo;
    int N, C, H, W, F, Ho, Wo;
    int LR, LY, RY, ipb, bpi, rows, pitch, cc, nchunks, nstage, fsets;
    int in_bytes, w_bytes, stage_bytes;
    int xoff; // smem column of image column 0 (the TMA box starts at column -xoff)
    // ordered stream-K (as kernel_pipe.cu): partial sums of split units, flags, tickets
    int sk;
    float2 *sk_part;              // [grid][8 warps][NACC][32 lanes]
    unsigned long long *sk_flag;  // [grid][8 warps]
    unsigned *sk_ticket;          // [2]
    unsigned long long epoch;
};

template <int S, bool FUSED>
__global__ void __launch_bounds__(32 * DW, 1) dense_kernel(const __grid_constant__ CUtensorMap tmap,
                                                          const DenseArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full_bar[DMAXSTAGE], empty_bar[DMAXSTAGE];
    __shared__ int done_cnt[DMAXSTAGE];
    // this CTA's work, in processing order: [head: unit uh, chunks [0, hj) -> park],
    // nf whole units, [tail: unit ut, chunks [tj, nchunks) -> resume, then store]
    struct Sched {
        int bid, uh, hj, nf, uf0, ut, tj, total;
    };
    __shared__ Sched sch;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ns = a.nstage;
    const uint32_t smem0 = smem_u32(smem);
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(smem_u32(&full_bar[s]), 1u);
            mbar_init(smem_u32(&empty_bar[s]), uint32_t(DW));
            done_cnt[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    const int nblocks = a.ipb > 1 ? (a.N + a.ipb - 1) / a.ipb : a.N * a.bpi;
    const int nunits = nblocks * a.fsets;
    const int nch = a.nchunks;
    if (threadIdx.x == 0) {
        Sched q{0, 0, 0, 0, 0, 0, 0, 0};
        if (a.sk) {
            // ordered stream-K: the CTA with arrival ticket b owns chunk steps
            // [b*T/G, (b+1)*T/G) of the unit sequence (see kernel_pipe.cu for why a
            // ticket rather than blockIdx.x)
            const int b = int(atomicAdd(a.sk_ticket, 1u));
            const int64_t T = int64_t(nunits) * nch;
            const int64_t s0 = T * b / gridDim.x, e0 = T * (b + 1) / gridDim.x;
            q.bid = b;
            if (e0 % nch) { q.uh = int(e0 / nch); q.hj = int(e0 % nch); }
            if (s0 % nch) { q.ut = int(s0 / nch); q.tj = int(s0 % nch); }
            q.uf0 = int((s0 + nch - 1) / nch);
            q.nf = int(e0 / nch) - q.uf0;
            q.total = q.hj + q.nf * nch + (q.tj ? nch - q.tj : 0);
        } else {
            q.bid = int(blockIdx.x);
            q.uf0 = q.bid;
            q.nf = q.bid < nunits ? (nunits - 1 - q.bid) / int(gridDim.x) + 1 : 0;
            q.total = q.nf * nch;
        }
        sch = q;
    }
    __syncthreads();
    // the ticket above comes from this launch's own counter slot; x and the parked
    // partials may only be read once the previous grid is complete
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const Sched sc = sch;
    auto full_unit = [&](int i) { return a.sk ? sc.uf0 + i : sc.uf0 + i * int(gridDim.x); };

    // stage kk of this CTA's sequence: the TMA box of its unit's rows x cc channels and
    // the weight slab of its channel set, on the stage's full barrier (one lane)
    auto fill = [&](int kk) {
        const int s = kk % ns;
        int u, j;
        if (kk < sc.hj) { u = sc.uh; j = kk; }
        else {
            const int k2 = kk - sc.hj;
            if (k2 < sc.nf * nch) { u = full_unit(k2 / nch); j = k2 % nch; }
            else { u = sc.ut; j = sc.tj + (k2 - sc.nf * nch); }
        }
        const int fs = u % a.fsets, blk = u / a.fsets;
        int n, iy;
        if (a.ipb > 1) { n = blk * a.ipb; iy = -1; }
        else { n = blk / a.bpi; iy = (blk % a.bpi) * a.LY * DT - 1; }
        const uint32_t fb = smem_u32(&full_bar[s]);
        const uint32_t dst = smem0 + uint32_t(s) * uint32_t(a.stage_bytes);
        // order the consumers' generic-proxy reads of this stage before the async writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(fb, uint32_t(a.ipb * a.cc * a.rows * a.pitch) * 4u + uint32_t(a.w_bytes));
        tma_load_4d(&tmap, fb, dst, -a.xoff, iy, j * a.cc, n);
        bulk_load(dst + uint32_t(a.in_bytes), a.wslab + (size_t(fs) * nch + j) * (a.w_bytes / 4),
                  uint32_t(a.w_bytes), fb);
    };
    if (threadIdx.x == 0)
        for (int kk = 0; kk < min(ns, sc.total); ++kk) fill(kk);

    // consumer lane -> (image slot, lane row in it, tile column)
    const int lx = lane % a.LR, ly = lane / a.LR;
    const int im = a.ipb > 1 ? ly / a.RY : 0;
    const int yl = a.ipb > 1 ? ly % a.RY : ly;
    const bool lane_ok = ly < a.LY && im < a.ipb;
    // word offset of this thread's window inside a stage's input box
    const int win = lane_ok ? (im * a.cc * a.rows + yl * DT) * a.pitch + S * lx + a.xoff - 1 : 0;
    const int ch_words = a.rows * a.pitch;
    constexpr int NACC = DR / 2 * DT * S; // float2 accumulators per thread

    const int nitems = (sc.hj > 0) + sc.nf + (sc.tj > 0);
    int kk = 0;
    for (int it = 0; it < nitems; ++it) {
        int u, j0 = 0, j1 = nch, kind = 0; // kind: 0 whole unit, 1 head (park), 2 tail (resume)
        if (sc.hj > 0 && it == 0) { u = sc.uh; j1 = sc.hj; kind = 1; }
        else {
            const int i2 = it - (sc.hj > 0);
            if (i2 < sc.nf) u = full_unit(i2);
            else { u = sc.ut; j0 = sc.tj; kind = 2; }
        }
        const int fs = u % a.fsets, blk = u / a.fsets;
        float2 acc[DR / 2][DT][S];
        if (kind == 2) {
            // resume: CTA b-1 parked this unit's partial sums (it did that first)
            const size_t slot = size_t(sc.bid - 1) * DW + warp;
            unsigned long long f;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(a.sk_flag + slot) : "memory");
            } while (f != a.epoch);
            const float2 *src = a.sk_part + slot * NACC * 32 + lane;
#pragma unroll
            for (int p = 0; p < DR / 2; ++p)
#pragma unroll
                for (int t = 0; t < DT; ++t)
#pragma unroll
                    for (int q = 0; q < S; ++q) acc[p][t][q] = __ldcg(src + size_t((p * DT + t) * S + q) * 32);
        } else {
#pragma unroll
            for (int p = 0; p < DR / 2; ++p)
#pragma unroll
                for (int t = 0; t < DT; ++t)
#pragma unroll
                    for (int q = 0; q < S; ++q) acc[p][t][q] = make_float2(0.0f, 0.0f);
        }

        for (int j = j0; j < j1; ++j, ++kk) {
            const int s = kk % ns, rnd = kk / ns;
            mbar_wait(smem_u32(&full_bar[s]), uint32_t(rnd & 1));
            const float *in = reinterpret_cast<const float *>(smem + size_t(s) * a.stage_bytes) + win;
            const float4 *wq = reinterpret_cast<const float4 *>(smem + size_t(s) * a.stage_bytes + a.in_bytes) +
                               size_t(warp) * a.cc * 9 * 2;
#pragma unroll 1
            for (int cl = 0; cl < a.cc; ++cl) {
                float xw[DT + 2][S + 2];
#pragma unroll
                for (int r = 0; r < DT + 2; ++r)
#pragma unroll
                    for (int q = 0; q < S + 2; ++q) xw[r][q] = in[cl * ch_words + r * a.pitch + q];
#pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                    const int ky = tap / 3, kx = tap % 3;
                    const float4 w0 = wq[(cl * 9 + tap) * 2], w1 = wq[(cl * 9 + tap) * 2 + 1];
                    const float2 wp[4] = {make_float2(w0.x, w0.y), make_float2(w0.z, w0.w),
                                          make_float2(w1.x, w1.y), make_float2(w1.z, w1.w)};
#pragma unroll
                    for (int t = 0; t < DT; ++t)
#pragma unroll
                        for (int q = 0; q < S; ++q) {
                            const float xv = xw[t + ky][q + kx];
                            const float2 xx = make_float2(xv, xv);
#pragma unroll
                            for (int p = 0; p < DR / 2; ++p) acc[p][t][q] = __ffma2_rn(xx, wp[p], acc[p][t][q]);
                        }
                }
            }
            // release stage s; the LAST warp to release it refills it with stage kk + ns
            // (no producer warp: a 9th warp would cap every thread at 168 registers)
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(smem_u32(&empty_bar[s]));
                const int old = atomicAdd(&done_cnt[s], 1);
                if (old == rnd * DW + DW - 1) {
                    mbar_wait(smem_u32(&empty_bar[s]), uint32_t(rnd & 1)); // acquire every warp's reads
                    if (kk + ns < sc.total) fill(kk + ns);
                }
            }
        }

        if (kind == 1) {
            // park: this warp's partial sums into slot (b, warp) for CTA b+1
            float2 *dst = a.sk_part + (size_t(sc.bid) * DW + warp) * NACC * 32 + lane;
#pragma unroll
            for (int p = 0; p < DR / 2; ++p)
#pragma unroll
                for (int t = 0; t < DT; ++t)
#pragma unroll
                    for (int q = 0; q < S; ++q) __stcg(dst + size_t((p * DT + t) * S + q) * 32, acc[p][t][q]);
            __threadfence();
            __syncwarp();
            if (lane == 0)
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.sk_flag + size_t(sc.bid) * DW + warp),
                             "l"(a.epoch)
                             : "memory");
            continue;
        }

        // epilogue (a6): + bias (one FP32 add); conv: [+ residual] [ReLU] and store the
        // lane's 2 x S pixels of its 8 channels; fused: ReLU, 2x2 max, first-max argmax
        int n, oy0;
        if (a.ipb > 1) { n = blk * a.ipb + im; oy0 = yl * DT; }
        else { n = blk / a.bpi; oy0 = (blk % a.bpi) * a.LY * DT + yl * DT; }
        const bool out_ok = lane_ok && n < a.N;
        if constexpr (!FUSED) {
            if (!out_ok) continue;
#pragma unroll
            for (int r = 0; r < DR; ++r) {
                const int f = fs * (DW * DR) + warp * DR + r;
                if (f >= a.F) continue;
                const float b = __ldg(a.bias + f);
                const size_t plane = ((size_t)n * a.F + f) * a.Ho * a.Wo;
                float *yp = a.y + plane;
#pragma unroll
                for (int t = 0; t < DT; ++t) {
                    const int oy = oy0 + t;
                    if (oy >= a.Ho) continue;
#pragma unroll
                    for (int q = 0; q < S; ++q) {
                        const int ox = S * lx + q;
                        if (ox < a.Wo) {
                            float v = __fadd_rn((r & 1) ? acc[r / 2][t][q].y : acc[r / 2][t][q].x, b);
                            if (a.epi & 2) v = __fadd_rn(v, a.res[plane + (size_t)oy * a.Wo + ox]);
                            if (a.epi & 1) v = v > 0.0f ? v : 0.0f;
                            yp[(size_t)oy * a.Wo + ox] = v;
                        }
                    }
                }
            }
        } else {
            // the lane's two rows are one pool row (oy0 is even); its columns S*lx ..
            // S*lx + S-1.  With S odd, a lane starting on an even column owns the pair
            // straddling into lane + 1 (whose first column arrives by shuffle); a lane
            // starting on an odd column leaves its first column to lane - 1.
            const int py = oy0 >> 1;
#pragma unroll
            for (int r = 0; r < DR; ++r) {
                const int f = fs * (DW * DR) + warp * DR + r;
                const float b = __ldg(a.bias + min(f, a.F - 1));
                float rl[DT][S + 1];
#pragma unroll
                for (int t = 0; t < DT; ++t) {
#pragma unroll
                    for (int q = 0; q < S; ++q) {
                        const float v = __fadd_rn((r & 1) ? acc[r / 2][t][q].y : acc[r / 2][t][q].x, b);
                        rl[t][q] = v > 0.0f ? v : 0.0f;
                    }
                    rl[t][S] = __shfl_down_sync(0xffffffffu, rl[t][0], 1);
                }
                if (!out_ok || f >= a.F || py >= a.Po) continue;
                float *yp = a.y + ((size_t)n * a.F + f) * a.Po * a.Qo + (size_t)py * a.Qo;
                int32_t *ap = a.argmax ? a.argmax + ((size_t)n * a.F + f) * a.Po * a.Qo + (size_t)py * a.Qo : nullptr;
                const int c0 = S * lx;
#pragma unroll
                for (int q0 = 0; q0 < S; ++q0) {
                    if (((c0 + q0) & 1) != 0) continue; // pools start on even columns
                    const int px = (c0 + q0) >> 1;
                    if (px >= a.Qo) continue;
                    float best = 0.0f;
                    int bidx = 0;
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const int dy = w >> 1, dx = w & 1;
                        const float rv = rl[dy][q0 + dx];
                        if (w == 0 || rv > best) {
                            best = rv;
                            bidx = (oy0 + dy) * a.Wo + c0 + q0 + dx;
                        }
                    }
                    yp[px] = best;
                    if (ap) ap[px] = bidx;
                }
            }
        }
    }
    if (a.sk) {
        // the last CTA to finish resets the arrival counters for the next launch
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(a.sk_ticket + 1, 1u) == gridDim.x - 1) {
                a.sk_ticket[0] = 0u;
                a.sk_ticket[1] = 0u;
                __threadfence();
            }
        }
    }
}

// Right-pads rows to Wq (multiple of 4 floats) so TMA can stage inputs whose row
// stride is not a multiple of 16 bytes: xp[row][ix] = x[row][ix] (ix < W), 0 beyond.
__global__ void __launch_bounds__(256) dense_pad_kernel(const float *__restrict__ x, float *__restrict__ xp,
                                                        int64_t rows, int W, int Wq) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * Wq;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / Wq;
        const int ix = int(i - row * Wq);
        xp[i] = ix < W ? __ldg(x + row * W + ix) : 0.0f;
    }
}

PFN_cuTensorMapEncodeTiled_v12000 dense_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// Bank-conflict degree of the LDS.32 window loads of one warp for a candidate pitch
// (32 lanes, one word each; distinct words sharing a bank serialise).
int dense_conflicts(const DenseGeometry &g, int pitch) {
    int worst = 1;
    for (int k = 0; k < g.S + 2; ++k) {
        int cnt[32] = {};
        for (int l = 0; l < 32; ++l) {
            const int lx = l % g.LR, ly = l / g.LR;
            const int im = g.ipb > 1 ? ly / g.RY : 0, yl = g.ipb > 1 ? ly % g.RY : ly;
            if (ly >= g.LY || im >= g.ipb) continue;
            const int w = (im * g.cc * g.rows + yl * DT) * pitch + g.S * lx + 3 + k;
            ++cnt[w & 31];
        }
        for (int b = 0; b < 32; ++b) worst = std::max(worst, cnt[b]);
    }
    return worst;
}

} // namespace

bool dense_stream_k(const Plan &p, int64_t nunits, int grid) {
    if (p.knobs.sk >= 0) return p.knobs.sk == 1 && nunits > grid;
    return nunits > grid && nunits % grid != 0 && nunits < 16 * int64_t(grid);
}

// Relative efficiency the dense kernel's geometry allows on this layer (1 = every lane
// tile full and every SM busy): the covered-pixel share of the lane tiles times the
// share of SMs a single round of units keeps busy (stream-K balances larger counts).
// AUTO's dense decision uses it (spconv_api.cu): measured dense efficiency 0.68-0.70 of
// peak on the c2 / c5 shapes (estimate 0.95) vs 0.51 on c4 (estimate 0.76).
double dense_expected_efficiency(const Plan &p, int N) {
    DenseGeometry g;
    dense_geometry(p, g);
    if (!g.ok) return 0.0;
    const double covered = g.ipb > 1 ? double(g.LY * g.LR) * DT * g.S                       // one unit
                                     : double(g.bpi) * g.LY * DT * g.LR * g.S;               // one image
    const double useful = g.ipb > 1 ? double(g.ipb) * p.Ho * p.Wo : double(p.Ho) * p.Wo;
    const int64_t blocks = g.ipb > 1 ? (N + g.ipb - 1) / g.ipb : int64_t(N) * g.bpi;
    const int64_t units = blocks * g.fsets;
    const int sms = sm_count_of_current_device();
    const double waves = units >= sms ? 0.95 : double(units) / sms;
    return useful / covered * waves;
}

bool dense_supported(int C, int H, int W, int F, int K, int stride, int pad) {
    (void)C; (void)H; (void)F;
    return K == 3 && stride == 1 && pad == 1 && W <= 224; // 32 lanes x 7 columns
}

void dense_geometry(const Plan &p, DenseGeometry &g) {
    g = DenseGeometry{};
    if (!dense_supported(p.C, p.H, p.W, p.F, p.K, p.stride, p.pad)) return;
    // lanes per row: the smallest power of two with ceil(Wo / LR) <= 8 columns per lane
    int LR = 1;
    while (LR < 32 && (p.Wo + LR - 1) / LR > 8) LR *= 2;
    const int need = (p.Wo + LR - 1) / LR;
    if (need > 8) return;
    g.S = need <= 7 ? 7 : 8;
    g.LR = LR;
    g.LY = 32 / LR;
    g.RY = (p.Ho + DT - 1) / DT;
    if (g.RY >= g.LY) {
        g.ipb = 1;
        g.bpi = (g.RY + g.LY - 1) / g.LY;
        g.rows = g.LY * DT + 2;
    } else {
        g.ipb = g.LY / g.RY;
        g.bpi = 1;
        g.rows = p.H + 2;
    }
    g.padded = (p.W * 4) % 16 != 0;
    g.wq = g.padded ? (p.W + 3) & ~3 : p.W;
    g.xoff = 4; // the box starts at column -4 (16-byte aligned TMA start)
    g.fsets = (p.F + DW * DR - 1) / (DW * DR);
    // channels per stage: ~40 KB of input box + weights, all stages in ~200 KB
    const int min_pitch = ((g.S * g.LR + 4 + 2) + 3) & ~3;
    const int per_ch = g.ipb * g.rows * (min_pitch + 32) * 4 + DW * 9 * DR * 4;
    // ~40 KB stages for <= 64 channels (finer chunks balance the stream-K split of the
    // few units such layers have: c2 shape 147 vs 150 us at 60 KB), ~60 KB above
    // (fewer stage turnovers: c5 shape 17.1 vs 18.1 ms) -- profiles/r02/dense_stage_ab.jsonl
    const int target = p.knobs.dense_stage > 0 ? p.knobs.dense_stage : (p.C <= 64 ? 40960 : 61440);
    g.cc = std::max(1, std::min(p.C, target / per_ch));
    for (int d = g.cc; d >= 1; --d) // a divisor of C close to cc (no zero-padded tail chunk)
        if (p.C % d == 0) {
            if (2 * d >= g.cc) g.cc = d;
            break;
        }
    g.nchunks = (p.C + g.cc - 1) / g.cc;
    int best = min_pitch, best_deg = 1 << 30;
    for (int cand = min_pitch; cand <= min_pitch + 28; cand += 4) {
        const int deg = dense_conflicts(g, cand);
        if (deg < best_deg) { best_deg = deg; best = cand; }
    }
    g.pitch = best;
    if (g.pitch > 256 || g.rows > 256 || g.cc > 256 || g.ipb > 256) return;
    g.in_bytes = (g.ipb * g.cc * g.rows * g.pitch * 4 + 127) & ~127;
    g.w_bytes = DW * g.cc * 9 * DR * 4;
    g.stage_bytes = (g.in_bytes + g.w_bytes + 127) & ~127;
    g.nstage = std::min(DMAXSTAGE, (200 * 1024) / g.stage_bytes);
    if (g.nstage < 2) return;
    g.smem_bytes = size_t(g.nstage) * g.stage_bytes;
    g.ok = true;
}

// The weight slab: [fset][chunk][warp][c in chunk][tap][8] floats, zero for absent taps
// (the densified CSR rows) and for channels / rows beyond C / F.
std::vector<float> dense_weights(const Plan &p, const DenseGeometry &g, const std::vector<int32_t> &rowptr,
                                 const std::vector<int32_t> &colidx, const std::vector<float> &values) {
    std::vector<float> w(size_t(g.fsets) * g.nchunks * DW * g.cc * 9 * DR, 0.0f);
    for (int f = 0; f < p.F; ++f) {
        const int fs = f / (DW * DR), wr = (f % (DW * DR)) / DR, r = f % DR;
        for (int32_t j = rowptr[size_t(f)]; j < rowptr[size_t(f) + 1]; ++j) {
            const int col = colidx[size_t(j)], c = col / 9, tap = col % 9;
            const int ch = c / g.cc, cl = c % g.cc;
            const size_t at = ((((size_t(fs) * g.nchunks + ch) * DW + wr) * g.cc + cl) * 9 + tap) * DR + r;
            w[at] = values[size_t(j)];
        }
    }
    return w;
}

cudaError_t launch_dense(const Plan &p, int N, const float *x, float *y, int32_t *argmax, bool fused,
                         cudaStream_t s, const float *res, int epi) {
    const DenseGeometry &g = p.dense_geo;
    if (!g.ok || !p.d_wdense || dense_encode() == nullptr) return cudaErrorInvalidConfiguration;
    float *xp = nullptr;
    const float *src = x;
    if (g.padded || (reinterpret_cast<uintptr_t>(x) & 15) != 0) {
        const size_t bytes = size_t(N) * p.C * p.H * g.wq * 4;
        keep_pool_cached();
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&xp), bytes, s);
        if (e != cudaSuccess) return e;
        const int64_t rows = int64_t(N) * p.C * p.H;
        const int blocks = int(std::min<int64_t>((rows * g.wq + 255) / 256, 148 * 16));
        dense_pad_kernel<<<blocks, 256, 0, s>>>(x, xp, rows, p.W, g.wq);
        if ((e = cudaGetLastError()) != cudaSuccess) {
            cudaFreeAsync(xp, s);
            return e;
        }
        src = xp;
    }
    DenseArgs a;
    a.x = src; a.bias = p.d_bias; a.wslab = p.d_wdense; a.y = y;
    a.res = res; a.argmax = argmax; a.epi = fused ? 0 : epi; a.Po = p.Ho / 2; a.Qo = p.Wo / 2;
    a.N = N; a.C = p.C; a.H = p.H; a.W = p.W; a.F = p.F; a.Ho = p.Ho; a.Wo = p.Wo;
    a.LR = g.LR; a.LY = g.LY; a.RY = g.RY; a.ipb = g.ipb; a.bpi = g.bpi; a.rows = g.rows; a.pitch = g.pitch;
    a.cc = g.cc; a.nchunks = g.nchunks; a.nstage = g.nstage; a.fsets = g.fsets;
    a.in_bytes = g.in_bytes; a.w_bytes = g.w_bytes; a.stage_bytes = g.stage_bytes; a.xoff = g.xoff;
    const int64_t nblocks = g.ipb > 1 ? (N + g.ipb - 1) / g.ipb : int64_t(N) * g.bpi;
    const int64_t nunits = nblocks * g.fsets;
    const int grid = int(std::min<int64_t>(nunits, sm_count_of_current_device()));
    const int wsrc = (src == x) ? p.W : g.wq;
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    Plan &mp = const_cast<Plan &>(p);
    const bool cached = mp.cache.find_map(src, N, &g, map);
    cuuint64_t dims[4] = {(cuuint64_t)wsrc, (cuuint64_t)p.H, (cuuint64_t)p.C, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)wsrc * 4, (cuuint64_t)p.H * wsrc * 4, (cuuint64_t)p.C * p.H * wsrc * 4};
    cuuint32_t box[4] = {(cuuint32_t)g.pitch, (cuuint32_t)g.rows, (cuuint32_t)g.cc, (cuuint32_t)g.ipb};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (!cached) {
        CUresult r = dense_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(src), dims,
                                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            if (xp) cudaFreeAsync(xp, s);
            return cudaErrorInvalidValue;
        }
        mp.cache.put_map(src, N, &g, map);
    }
    // ordered stream-K when the units do not divide evenly over the persistent CTAs
    // (c2 shape: 224 units on 148 SMs would leave the second round a third full)
    a.sk = dense_stream_k(p, nunits, grid) ? 1 : 0;
    a.sk_part = nullptr; a.sk_flag = nullptr; a.sk_ticket = nullptr; a.epoch = 0;
    SkWorkspace skws;
    if (a.sk) {
        const size_t part_bytes = size_t(grid) * DW * (DR / 2 * DT * g.S) * 32 * sizeof(float2);
        cudaError_t e = stream_k_workspace(p, s, part_bytes, grid * DW, skws);
        if (e != cudaSuccess) {
            if (xp) cudaFreeAsync(xp, s);
            return e;
        }
        a.sk_part = reinterpret_cast<float2 *>(skws.part);
        a.sk_flag = skws.flag;
        a.sk_ticket = skws.ticket;
        a.epoch = next_sk_epoch();
    }
    cudaError_t err;
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(grid));
        cfg.blockDim = dim3(32u * DW);
        cfg.dynamicSmemBytes = g.smem_bytes;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = p.knobs.pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        auto go = [&](auto kern) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(g.smem_bytes));
            return e == cudaSuccess ? cudaLaunchKernelEx(&cfg, kern, map, a) : e;
        };
        if (g.S == 7) err = fused ? go(dense_kernel<7, true>) : go(dense_kernel<7, false>);
        else err = fused ? go(dense_kernel<8, true>) : go(dense_kernel<8, false>);
    }
    {
        cudaError_t e2 = skws.release(s);
        if (err == cudaSuccess) err = e2;
    }
    if (xp) {
        cudaError_t e2 = cudaFreeAsync(xp, s);
        if (err == cudaSuccess) err = e2;
    }
    return err;
}

} // namespace spconv
