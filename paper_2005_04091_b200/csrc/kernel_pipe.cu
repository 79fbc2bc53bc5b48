// kernel_pipe.cu — warp-specialised, TMA-pipelined CSR sparse direct
// convolution for sm_100a (K = 3, stride 1, pad 1: the ResNet/VGG layers of
// BASELINE.json), with the conv-only and the fused bias+ReLU+2x2-maxpool
// epilogues.  This is the v2 ("pipe") kernel; kernel_tiled.cu is v1.
//
// What it computes is PAPER.md L393-401 (per output channel, per nonzero j of
// its CSR row: out[n][y][x] += value[j] * in[...offset(colidx[j])]) under the
// FP32 contract of include/spconv.h (ascending colidx, fma, bias after the
// sum), so the result is bit-identical to the oracle.  How it maps to B200:
//
//  * CTA = GPC warps (<= 8, so 2 warps per SM sub-partition and up to 255
//    registers each).  Warp w owns row
//    group g = gset*GPC + w (R output channels with balanced nnz, SURVEY.md
//    §8(a) a3; "register blocking"); lane l owns one 4x4
//    output tile, so a thread accumulates R x 4 x 4 outputs in registers
//    (64-bit pairs: packed FFMA2).  All warps of a CTA share the pixel block.
//  * Staging (a4; "data prefetching"): one input channel per
//    stage of an NSTAGE-deep shared-memory ring, filled with (i) the block's
//    input rows + halo via one 4-D TMA tile load whose out-of-bounds zero
//    fill is the padding (cp.async with zero fill when the TMA stride rule
//    fails), and (ii) the CTA's decoded tap stream for that channel via one
//    bulk copy, completing on the stage's "full" mbarrier.  There is no
//    producer warp and no __syncthreads in the main loop: the LAST warp to
//    finish with a stage (shared-memory counter) refills it, so no warp ever
//    waits for a slower one except on data.
//  * Consumer (a5): per channel, load the 6x6 window (LDS.128 + LDS.64 per
//    row), then run the threaded-code dispatcher of dispatch2_gen.inc over
//    the warp's entries {v, next case}: one brx.idx per nonzero, the jump
//    target of nonzero k+1 and the entry of k+2 fetched while k's FMAs issue.
//  * Epilogue (a6): + bias and store; or ReLU, 2x2 max and first-max argmax
//    (the conv output is never written).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "async_copy.cuh"
#include "spconv_internal.h"

namespace spconv {
namespace {

constexpr int MAXSTAGE = 8;
constexpr int MAX_GPC = 8;
// R = 2 (DESIGN.md §7 "next" 1): half the accumulators, so 12 warps fit the register
// file (<= 168 registers per thread) -- more warps to hide the per-nonzero dispatch
constexpr int MAX_GPC_R2 = 12;

struct PipeArgs {
    const float *x;
    const float *res; // residual added before the optional ReLU (EPI & 2), may alias y
    float *y;
    int32_t *argmax;
    const float *bias;
    const int32_t *group_rows;
    const int32_t *chunk_start; // byte offsets of (gset, c) chunks in stream
    const char *stream;
    int N, C, H, W, F, Ho, Wo, Po, Qo;
    int xs, tiles_x, tiles_y, ipb, tr, lanes, blocks_y, rs, pitch, nstage, in_words, in_pad, st_bytes;
    // wide rows: the row is split into colblocks column blocks of cb_tiles tiles (units of
    // their own); each block's lanes cover one extra tile (tiles_x = cb_tiles + 1) whose
    // outputs belong to the next block -- computed, not stored, it feeds the fused
    // epilogue's pool pairs that straddle the block boundary
    int colblocks, cb_tiles, tiles_total;
    int cc, nchunks;
    int band; // 1: the ipb slots of a unit are tile-row bands of the flattened (image, tile row) sequence
    uint32_t lane_map[32]; // per lane: slot << 16 | tile row << 8 | tile column (lane_tile on the host)
    int gpc, num_groups, num_gsets;
    int tma;
    int ent; // == 8, the tap-stream entry stride: a runtime value so ptxas cannot fold it (SPC2_ENT_REG)
    // ordered stream-K (sk = 1): CTA b owns the contiguous chunk range
    // [b*U*nch/grid, (b+1)*U*nch/grid) of the U units; a unit cut by a range end is
    // started by CTA b (its "head", done FIRST, accumulators parked in sk_part slot b)
    // and finished by CTA b+1 (its "tail", done LAST, continuing from the parked
    // accumulators), so every output is still one ascending fma chain (FP32 contract).
    int sk;
    ulonglong2 *sk_part;              // [grid][gpc][R*PT*PS/4][32 lanes]
    unsigned long long *sk_flag;      // [grid][gpc]: == epoch when slot (b, warp) is ready
    unsigned *sk_ticket;              // [2]: arrival ticket, finished CTAs (0 between launches)
    unsigned long long epoch;
    unsigned long long *trace; // debug (SPCONV_PIPE_TRACE): per CTA 8 timestamps, or null
    int rev;                   // debug (SPCONV_PIPE_REV=1): CTA b does the work of CTA grid-1-b
    unsigned long long *prof;  // diagnostic builds (-DSPC_PROF): per-phase clock sums, or null
    // per-warp split points (sk_tab = 1; sk_split on the host): boundary b of the
    // contiguous ranges lies in unit sk_unit[b], at channel sk_ch[b][w] for warp w --
    // each warp's range then costs the same (its group's taps and reloads), which the
    // uniform channel split (sk_tab = 0) does not give
    int sk_tab;
    int32_t sk_unit[kSkTabCta + 1];
    uint16_t sk_ch[(kSkTabCta + 1) * kSkTabGpc];
};

using namespace dev; // mbarrier / TMA / bulk-copy wrappers (async_copy.cuh)

// Lane -> (image / band slot, tile row in it, tile column).  order 0: slot-major;
// order 1: tile-row-major (small images, several per unit: the lanes of a quarter-warp
// then span two slots, whose offset the pitch search can place on the other half of
// the shared-memory banks).  The column is always fastest, so lane + 1 is the next
// tile of the same row (the fused epilogue's shuffle relies on it).
inline void lane_tile(int li, int order, int ipb, int tr, int tiles_x, int &im, int &tyl, int &tx) {
    if (order == 0) {
        const int per_img = tr * tiles_x;
        im = li / per_img;
        const int rem = li - im * per_img;
        tyl = rem / tiles_x;
        tx = rem - tyl * tiles_x;
    } else {
        const int per_row = ipb * tiles_x;
        tyl = li / per_row;
        const int rem = li - tyl * per_row;
        im = rem / tiles_x;
        tx = rem - im * tiles_x;
    }
}

__device__ __forceinline__ float lo_f(uint64_t v) { return __uint_as_float(uint32_t(v)); }
__device__ __forceinline__ float hi_f(uint64_t v) { return __uint_as_float(uint32_t(v >> 32)); }

#define SPC2_ENT_REG (a.ent)
#include "dispatch2_gen.inc"

// Mask dispatcher (SPCONV_PIPE_DISPATCH=mask; the brx.idx walk is the default,
// measured faster on B200 -- DESIGN.md §7): per (row group, channel) the stream holds a 9*R-bit
// mask (bit tap*R + r: row r of the group has a nonzero at tap = ky*3 + kx) and a
// dense block of 9*R (v, v) value pairs (zero where the mask bit is clear).  The
// walk (SPC2_MASKWALK_*, gen_dispatch2.py) is straight-line code over the 9*R
// (tap, row) blocks with warp-uniform forward skips: no indirect branch and no
// jump-table load per nonzero, and the values of tap t+1 are loaded at static
// offsets while tap t runs.  Within a row the taps are consumed in ascending
// (ky, kx) order and channels ascend, i.e. ascending colidx (the FP32 contract;
// a skipped tap contributes exactly nothing, as fma(0, x, acc) == acc).
// Segment layout per (warp, stage): the ncl masks (16-byte padded), then the ncl
// dense value blocks back to back.
template <int R, int PT, int PS>
__device__ __forceinline__ void mask_walk(uint64_t (&acc)[R][PT][PS / 2], const unsigned char *wbase,
                                          const unsigned char *seg, uint32_t seg_s, int ncl, int cl0, int cl1,
                                          uint32_t row_bytes, uint32_t ch_bytes) {
    // channels [cl0, cl1) of the ncl staged ones (a stream-K head / tail may cover part of a stage)
    constexpr int PAIRS = (PS + 2) / 2;
    const uint64_t *masks = reinterpret_cast<const uint64_t *>(seg);
    const uint32_t dense0 = uint32_t((ncl * 8 + 15) & ~15) + uint32_t(cl0) * 9u * R * 8u; // 16-byte aligned blocks
    uint32_t vb = seg_s + dense0;
    uint64_t v0[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v0[r] = *reinterpret_cast<const uint64_t *>(seg + dense0 + 8 * r);
#pragma unroll 1
    for (int cl = cl0; cl < cl1; ++cl) {
        uint64_t xw[PT + 2][PAIRS];
        const unsigned char *wptr = wbase + cl * ch_bytes;
#pragma unroll
        for (int i = 0; i < PT + 2; ++i) {
#pragma unroll
            for (int q = 0; q + 1 < PAIRS; q += 2) {
                const ulonglong2 v2 = *reinterpret_cast<const ulonglong2 *>(wptr + i * row_bytes + 16 * (q / 2));
                xw[i][q] = v2.x;
                xw[i][q + 1] = v2.y;
            }
            if constexpr (PAIRS % 2)
                xw[i][PAIRS - 1] = *reinterpret_cast<const uint64_t *>(wptr + i * row_bytes + 8 * (PAIRS - 1));
        }
        // broadcast from lane 0 so ptxas can prove the mask (and every branch on it)
        // warp-uniform: uniform branches need no convergence barriers
        const uint64_t m = __shfl_sync(0xffffffffu, masks[cl], 0);
        static_assert(R == 4 && PT == 8 && PS == 4, "no mask walk generated for this variant");
        SPC2_MASKWALK_M4T8S4(acc, v0, xw, m, vb);
        vb += 9u * R * 8u;
    }
}

// Index of the k-th (1-based) entry of a warp's stream segment whose case field
// is the "next channel" marker (case id `marker`).  Entries are 8-byte {v, case of
// the following entry} behind a lead entry, so that index is the entry BEFORE the
// marker: setting its case field to "end" ends the walk after channel k-1, and the
// marker entry (index + 1) is a valid lead entry for a walk starting at channel k.
// Warp-cooperative (ballot over 32 entries at a time); the caller asks for k < the
// stage's channel count, so the marker exists.
// brx.idx streams: markers (entry j + 1 when seg[j].y == marker) advance the window by
// k channels (k = the marker entry's value field).  Returns the j of the first marker
// whose target channel (running sum of the advances) is >= cl, with *target set, or
// the j whose .y is the end case (marker + 1) when no later marker reaches cl
// (*target = -1).  Warp-collective.
// Reads only the warp's own segment (nent entries): never past the stage's stream
// chunk, never another warp's segment (which that warp may be patching).
__device__ __forceinline__ int find_channel(const uint2 *seg, int nent, int cl, int lane, uint32_t marker,
                                            int *target) {
    int run = 0;
    for (int base = 0;; base += 32) {
        const uint2 e = base + lane < nent ? seg[base + lane] : make_uint2(0u, 0u);
        const bool mk = e.y == marker, en = e.y == marker + 1u;
        uint32_t nx = __shfl_down_sync(0xffffffffu, e.x, 1);
        if (lane == 31 && mk) nx = base + 32 < nent ? seg[base + 32].x : 0u;
        int sc = mk ? int(nx) : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, sc, o);
            if (lane >= o) sc += t;
        }
        const unsigned m = __ballot_sync(0xffffffffu, (mk && run + sc >= cl) || en);
        if (m) {
            const int l = __ffs(m) - 1;
            const int t = __shfl_sync(0xffffffffu, run + sc, l);
            const bool isend = __shfl_sync(0xffffffffu, en ? 1 : 0, l) != 0;
            *target = isend ? -1 : t;
            return base + l;
        }
        run += __shfl_sync(0xffffffffu, sc, 31);
    }
}

// Fill stage s with chunk k (channels [k*cc, k*cc + cc)) of the unit at (n0, iy0)
// and the unit's stream chunk [c_beg, c_end).  TMA: called by one lane.
// cp.async: called by a whole warp.
template <int XS, int STG>
__device__ __forceinline__ void fill_stage(const CUtensorMap *tmap, const PipeArgs &a, uint32_t smem0,
                                           uint32_t fb, int s, int k, int n0, int iy0, int x0, int c_beg,
                                           int c_end, int lane) {
    const uint32_t stage_bytes = uint32_t(a.in_pad + a.st_bytes);
    const uint32_t dst_in = smem0 + uint32_t(s) * stage_bytes;
    const uint32_t dst_st = dst_in + uint32_t(a.in_pad);
    const uint32_t st_bytes = uint32_t(c_end - c_beg);
    // order the consumers' generic-proxy reads of this stage before the async-proxy writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if constexpr (STG == 1) {
        // TMA: XS == 3 loads the caller's tensor from ix = -4 (16-byte aligned start);
        // XS == 0 loads the left-padded copy (column 0 = the zero pad) from column 0
        mbar_expect_tx(fb, uint32_t(a.in_words) * 4u + st_bytes);
        if (a.band) {
            // one box per band: [cc][PT + 2][pitch] of image n from row ty*PT - 1
            const int nb = a.N * a.tiles_y;
            const uint32_t slot_bytes = uint32_t(a.cc * a.rs * a.pitch) * 4u;
            for (int b = 0; b < a.ipb; ++b) {
                const int v = min(n0 + b, nb - 1); // a ragged last unit reloads the last band (not stored)
                const int n = v / a.tiles_y, ty = v - n * a.tiles_y;
                tma_load_4d(tmap, fb, dst_in + uint32_t(b) * slot_bytes, x0 + (XS == 3 ? -4 : 0),
                            ty * (a.rs - 2) - 1, k * a.cc, n);
            }
        } else {
            tma_load_4d(tmap, fb, dst_in, x0 + (XS == 3 ? -4 : 0), iy0, k * a.cc, n0);
        }
        bulk_load(dst_st, a.stream + c_beg, st_bytes, fb);
    } else {
        if (lane == 0) {
            mbar_expect_tx(fb, st_bytes);
            bulk_load(dst_st, a.stream + c_beg, st_bytes, fb);
        }
        // smem layout of a stage = the TMA box order [image][channel][row][col]
        const int per_ch = a.rs * a.pitch, per_img = a.cc * per_ch;
        for (int e = lane; e < a.in_words; e += 32) {
            const int im = e / per_img;
            int rem = e - im * per_img;
            const int cl = rem / per_ch;
            rem -= cl * per_ch;
            const int r = rem / a.pitch, col = rem - r * a.pitch;
            int n = n0 + im, iyb = iy0;
            if (a.band) {
                const int v = n0 + im;
                n = v / a.tiles_y;
                iyb = (v - n * a.tiles_y) * (a.rs - 2) - 1;
            }
            const int c = k * a.cc + cl, iy = iyb + r, ix = x0 + col - (XS + 1);
            const bool ok = n < a.N && c < a.C && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
            const float *src = ok ? a.x + (((size_t)n * a.C + c) * a.H + iy) * a.W + ix : a.x;
            cp_async_4(dst_in + uint32_t(e) * 4u, src, ok);
        }
        cp_async_arrive_noinc(fb);
    }
}

// A unit of work = (image group, block of tile rows, group set): decoded here.
struct Unit {
    int gs, n0, ty0, cb;
};
template <bool CB>
__device__ __forceinline__ Unit decode_unit(const PipeArgs &a, int u) {
    Unit r;
    r.gs = u % a.num_gsets;
    u /= a.num_gsets;
    r.cb = 0;
    if constexpr (CB) {
        r.cb = u % a.colblocks;
        u /= a.colblocks;
    }
    if (a.band) { // n0 = first band of the unit
        r.ty0 = 0;
        r.n0 = u * a.ipb;
        return r;
    }
    r.ty0 = (u % a.blocks_y) * a.tr;
    r.n0 = (u / a.blocks_y) * a.ipb;
    return r;
}

// EPI (conv-only path): bit 0 = ReLU, bit 1 = add a residual tensor; the order is
// y = ReLU((acc + bias) + residual), two FP32 adds (reading for NEXT-3).
// EPI bit 2 (any path): wide rows in column blocks (PipeGeometry::colblocks > 1) --
// a compile-time switch so the common kernels carry none of its index arithmetic.
template <int R, int PT, int PS, bool FUSED, int XS, int DISP, int STG, int EPI>
__global__ void __launch_bounds__(R == 2 ? 32 * MAX_GPC_R2 : 32 * MAX_GPC, 1)
    pipe_kernel(const __grid_constant__ CUtensorMap tmap, const PipeArgs a) {
    constexpr bool CB = (EPI & 4) != 0;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full_bar[MAXSTAGE], empty_bar[MAXSTAGE];
    __shared__ int done_cnt[MAXSTAGE];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
#ifdef SPC_PROF
    // diagnostic: clock cycles per phase, summed over warps: [0] other (prologue, loop
    // overhead), [1] waiting for a stage, [2] the tap walk, [3] stage release and refill,
    // [4] epilogue and the next unit's setup, [5] stream-K park, [6] stream-K resume
    // (wait + partials), [7] end-of-kernel barrier, [8] prologue (to the first stage wait)
    __shared__ unsigned long long s_prof[9];
    if (threadIdx.x < 9) s_prof[threadIdx.x] = 0;
    __syncthreads();
    unsigned prof_t = (unsigned)clock();
    int prof_ph = 8;
#define SPC_PROF_MARK(next)                                                    \
    do {                                                                      \
        const unsigned t_ = (unsigned)clock();                                \
        if (lane == 0) atomicAdd(&s_prof[prof_ph], (unsigned long long)(t_ - prof_t)); \
        prof_t = t_;                                                          \
        prof_ph = (next);                                                     \
    } while (0)
#else
#define SPC_PROF_MARK(next) do { } while (0)
#endif
    const int ns = a.nstage;
    unsigned long long *tr = a.trace ? a.trace + size_t(blockIdx.x) * 8 : nullptr;
    if (tr && threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        tr[0] = gtimer();
        tr[7] = smid;
    }
    const uint32_t stage_bytes = uint32_t(a.in_pad + a.st_bytes);
    const uint32_t smem0 = smem_u32(smem);
    // chunk byte offsets of every group set, the group -> output channel table and
    // the bias, copied once to shared memory (the epilogue must not wait on L2)
    int32_t *s_cstart = reinterpret_cast<int32_t *>(smem + size_t(ns) * stage_bytes);
    const int ncs = a.num_gsets * (a.nchunks + 1);
    int32_t *s_rows = s_cstart + ncs;
    float *s_bias = reinterpret_cast<float *>(s_rows + a.num_groups * R);

    // persistent CTA: units blockIdx.x, blockIdx.x + gridDim.x, ...; stages are
    // numbered across units so the ring prefetches the next unit's first channels
    // while this unit finishes (and during its epilogue).
    const int nunits = (a.band ? (a.N * a.tiles_y + a.ipb - 1) / a.ipb : ((a.N + a.ipb - 1) / a.ipb) * a.blocks_y) *
                       (CB ? a.colblocks : 1) * a.num_gsets;
    const int nch = a.nchunks;
    // this CTA's work items, in processing order: [head of unit uh: channels [0, hc),
    // chunks [0, hA)], nf whole units, [tail of unit ut: channels [tcs, C), chunks
    // [tc0, nch)].  Stream-K ranges are counted in input channels, so a split can fall
    // inside a stage: the head walks only the first channels of its last stage, the
    // tail starts its first stage part-way (find_channel).
    // The schedule lives in shared memory and is re-read where needed: values kept
    // in registers across the dispatcher's asm would cost it registers (measured: one
    // extra MOV on every case's jump-target path, -4% on c5).

    for (int i = threadIdx.x; i < ncs; i += blockDim.x) s_cstart[i] = __ldg(a.chunk_start + i);
    for (int i = threadIdx.x; i < a.num_groups * R; i += blockDim.x) s_rows[i] = __ldg(a.group_rows + i);
    for (int i = threadIdx.x; i < a.F; i += blockDim.x) s_bias[i] = __ldg(a.bias + i);
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) {
            mbar_init(smem_u32(&full_bar[s]), STG == 1 ? 1u : 33u);
            mbar_init(smem_u32(&empty_bar[s]), uint32_t(nwarps));
            done_cnt[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // Programmatic dependent launch: let the next launch on the stream start its
    // prologue on SMs this grid frees; griddepcontrol.wait (below, after the schedule)
    // waits for the previous grid.  Without the launch attribute both are no-ops.
    // Only plan tables (immutable) and this launch's counter slot are touched before.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    struct Sched {
        int hA, uh, tc0, tC, ut, nf, uf0, hc, tcs, total;
    };
    __shared__ Sched sch;
    __shared__ int s_bid;
    if (threadIdx.x == 0) {
        // work index.  Stream-K: an arrival ticket from this launch's counter slot
        // (stream_k_workspace: never shared with the launch this one overlaps, so it
        // can be taken before griddepcontrol.wait): CTA b's tail waits only for the
        // head of ticket b-1, whose CTA is already running, so the wait cannot depend
        // on a CTA that is not resident (MPS, green contexts, concurrent kernels).
        const int t = a.sk ? int(atomicAdd(a.sk_ticket, 1u)) : int(blockIdx.x);
        const int bid = a.rev ? int(gridDim.x) - 1 - t : t;
        s_bid = bid;
        if (tr) tr[5] = (unsigned long long)bid;
        Sched q{0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (a.sk && a.sk_tab) {
            // CTA-level structure from the per-warp table: a tail when any warp starts
            // inside unit sk_unit[bid], a head when any warp ends inside sk_unit[bid+1];
            // the stages cover the union of the warps' channel ranges
            const int C = a.C;
            const int u0 = a.sk_unit[bid], u1 = a.sk_unit[bid + 1];
            int mx0 = 0, mn0 = C, mx1 = 0;
            for (int w = 0; w < a.gpc; ++w) {
                const int c0 = a.sk_ch[bid * kSkTabGpc + w], c1 = a.sk_ch[(bid + 1) * kSkTabGpc + w];
                mx0 = max(mx0, c0);
                mn0 = min(mn0, c0);
                mx1 = max(mx1, c1);
            }
            if (mx0 > 0) { q.tcs = mn0; q.ut = u0; q.tc0 = mn0 / a.cc; q.tC = nch - q.tc0; }
            if (mx1 > 0) { q.hc = mx1; q.uh = u1; q.hA = (mx1 + a.cc - 1) / a.cc; }
            q.uf0 = u0 + (mx0 > 0 ? 1 : 0);
            q.nf = u1 - q.uf0;
        } else if (a.sk) {
            const int C = a.C;
            const int64_t tot = int64_t(nunits) * C;
            const int64_t s0 = tot * bid / gridDim.x, e0 = tot * (bid + 1) / gridDim.x;
            if (e0 % C) { q.hc = int(e0 % C); q.uh = int(e0 / C); q.hA = (q.hc + a.cc - 1) / a.cc; }
            if (s0 % C) { q.tcs = int(s0 % C); q.ut = int(s0 / C); q.tc0 = q.tcs / a.cc; q.tC = nch - q.tc0; }
            q.uf0 = int((s0 + C - 1) / C);
            q.nf = int(e0 / C) - q.uf0;
        } else {
            q.uf0 = bid;
            q.nf = bid < nunits ? (nunits - 1 - bid) / int(gridDim.x) + 1 : 0;
        }
        q.total = q.hA + q.nf * nch + q.tC;
        sch = q;
    }
    __syncthreads();
    // the previous grid (whose outputs x may be, and whose stream-K workspace this
    // launch reuses) must be complete before x or the parked partials are read
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int bid = s_bid;
    const int &hA = sch.hA, &uh = sch.uh, &tc0 = sch.tc0, &tC = sch.tC, &ut = sch.ut, &nf = sch.nf,
              &uf0 = sch.uf0, &hc = sch.hc, &tcs = sch.tcs, &total = sch.total;
    auto full_unit = [&](int j) { return a.sk ? uf0 + j : uf0 + j * int(gridDim.x); };

    auto fill = [&](int kk, int s) {
        int u, ch;
        if (kk < hA) {
            u = uh; ch = kk;
        } else {
            const int k2 = kk - hA, j = k2 / nch;
            if (j < nf) { u = full_unit(j); ch = k2 - j * nch; }
            else { u = ut; ch = tc0 + (k2 - nf * nch); }
        }
        const Unit un = decode_unit<CB>(a, u);
        const int32_t *cs = s_cstart + un.gs * (a.nchunks + 1);
        fill_stage<XS, STG>(&tmap, a, smem0, smem_u32(&full_bar[s]), s, ch, un.n0, un.ty0 * PT - 1,
                            CB ? un.cb * a.cb_tiles * PS : 0, cs[ch],
                       cs[ch + 1], lane);
    };
    if (warp == 0) {
        for (int kk = 0; kk < min(ns, total); ++kk) {
            if (STG == 1 && lane != 0) continue;
            fill(kk, kk);
        }
    }

    const bool lane_ok = lane < a.lanes;
    // (slot, tile row, tile column) of this lane, decomposed on the host (lane_tile)
    const uint32_t lm = a.lane_map[lane_ok ? lane : 0];
    const int im = int(lm >> 16), tyl = int((lm >> 8) & 0xff), tx = int(lm & 0xff);
    // byte offset of this thread's window inside a stage (16-byte aligned)
    const uint32_t win_off = uint32_t((im * a.cc * a.rs + tyl * PT) * a.pitch + tx * PS) * 4u;
    const uint32_t row_bytes = uint32_t(a.pitch) * 4u;
    const uint32_t ch_bytes = uint32_t(a.rs * a.pitch) * 4u;

    constexpr int SH = PS / 2, PAIRS = (PS + 2) / 2;
    static_assert(SH % 2 == 0, "partials are parked as 16-byte pairs");
    const int nitems = (hA > 0) + nf + (tC > 0);
    // ring position, kept incrementally (no integer division per stage):
    // kk = chunk sequence number, s = kk % ns, rnd = kk / ns
    int kk = 0, s = 0, rnd = 0;
    for (int it = 0; it < nitems; ++it) {
        int u, c0 = 0, kind = 0; // kind: 0 whole unit, 1 head (park), 2 tail (resume)
        if (hA > 0 && it == 0) {
            u = uh; kind = 1;
        } else {
            const int j = it - (hA > 0);
            if (j < nf) u = full_unit(j);
            else { u = ut; c0 = tc0; kind = 2; }
        }
        const int c1 = kind == 1 ? hA : nch;
        const Unit un = decode_unit<CB>(a, u);
        const int g = un.gs * a.gpc + warp;
        const bool active = g < a.num_groups; // warp-uniform

        uint64_t acc[R][PT][SH];
        if (kind == 2 && active) {
            SPC_PROF_MARK(6);
            // resume: wait for CTA b-1's parked accumulators of this warp (it parked
            // them before any other work, so this wait is normally already satisfied)
            const size_t slot = size_t(bid - 1) * a.gpc + warp;
            if (tr && threadIdx.x == 0) tr[3] = gtimer();
            unsigned long long f;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(a.sk_flag + slot) : "memory");
            } while (f != a.epoch);
            const ulonglong2 *src = a.sk_part + slot * (R * PT * SH / 2) * 32 + lane;
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int t = 0; t < PT; ++t)
#pragma unroll
                    for (int h = 0; h < SH; h += 2) {
                        const ulonglong2 v2 = __ldcg(src + size_t(((r * PT + t) * SH + h) / 2) * 32);
                        acc[r][t][h] = v2.x;
                        acc[r][t][h + 1] = v2.y;
                    }
            __syncwarp();
            if (tr && threadIdx.x == 0) tr[4] = gtimer();
            if (lane == 0) a.sk_flag[slot] = 0ull; // consumed (graph replays reuse the epoch)
            SPC_PROF_MARK(4);
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int t = 0; t < PT; ++t)
#pragma unroll
                    for (int h = 0; h < SH; ++h) acc[r][t][h] = 0ull;
        }

        for (int ch = c0; ch < c1; ++ch) {
            SPC_PROF_MARK(1);
            mbar_wait(smem_u32(&full_bar[s]), rnd & 1);
            SPC_PROF_MARK(2);
            if (active) {
                const unsigned char *stage = smem + size_t(s) * stage_bytes;
                const uint32_t st_base = smem0 + uint32_t(s) * stage_bytes + uint32_t(a.in_pad);
                const uint32_t seg_off = reinterpret_cast<const uint32_t *>(stage + a.in_pad)[warp];
                // channels [cl0, cl1) of this stage: all of them except at a stream-K split
                const int ncl = min(a.cc, a.C - ch * a.cc);
                int cl0 = 0, cl1 = ncl;
                if (kind == 1) { // head: channels [0, this warp's split)
                    const int h = a.sk_tab ? int(a.sk_ch[(bid + 1) * kSkTabGpc + warp]) : hc;
                    cl1 = min(ncl, max(0, h - ch * a.cc));
                }
                if (kind == 2) { // tail: channels [this warp's split, C)
                    const int t = a.sk_tab ? int(a.sk_ch[bid * kSkTabGpc + warp]) : tcs;
                    cl0 = min(ncl, max(0, t - ch * a.cc));
                }
                if (cl0 < cl1) { // (a warp's own split may leave it nothing in this stage)
                if constexpr (DISP == 1) {
                    mask_walk<R, PT, PS>(acc, stage + win_off, stage + a.in_pad + seg_off, st_base + seg_off, ncl,
                                         cl0, cl1, row_bytes, ch_bytes);
                } else {
                uint32_t sp = st_base + seg_off;
                uint32_t wp = smem0 + uint32_t(s) * stage_bytes + win_off; // first channel's window
                uint64_t xw[PT + 2][PAIRS];
                const unsigned char *wptr = stage + win_off;
                if (cl0 > 0 || cl1 < ncl) { // warp-uniform, at most twice per CTA
                    uint2 *seg = reinterpret_cast<uint2 *>(smem + size_t(s) * stage_bytes + a.in_pad + seg_off);
                    // this warp's segment ends at the next warp's header offset (or the chunk end)
                    const int32_t *csx = s_cstart + un.gs * (a.nchunks + 1);
                    const uint32_t seg_end = warp + 1 < a.gpc
                                                 ? reinterpret_cast<const uint32_t *>(stage + a.in_pad)[warp + 1]
                                                 : uint32_t(csx[ch + 1] - csx[ch]);
                    const int nent = int(seg_end - seg_off) / 8;
                    if (cl1 < ncl) {
                        // end the walk before channel cl1: the first marker reaching it becomes
                        // "end" (this warp's private copy of the segment; the refill overwrites it)
                        int t;
                        const int j = find_channel(seg, nent, cl1, lane, 9u * R, &t);
                        if (lane == 0 && t >= 0) seg[j].y = 9u * R + 1u;
                        __syncwarp();
                    }
                    if (cl0 > 0) {
                        // start at channel cl0: the first marker reaching it is the lead entry
                        // and the window starts at its target (channels cl0..t-1 hold no
                        // nonzeros of this group); none -> start at the end entry
                        int t;
                        const int j = find_channel(seg, nent, cl0, lane, 9u * R, &t);
                        if (t >= 0) {
                            sp += uint32_t(j + 1) * 8u;
                            wp += uint32_t(t) * ch_bytes;
                            wptr += size_t(t) * ch_bytes;
                        } else {
                            sp += uint32_t(j) * 8u;
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < PT + 2; ++i) {
#pragma unroll
                    for (int q = 0; q + 1 < PAIRS; q += 2) {
                        const ulonglong2 v2 =
                            *reinterpret_cast<const ulonglong2 *>(wptr + i * row_bytes + 16 * (q / 2));
                        xw[i][q] = v2.x;
                        xw[i][q + 1] = v2.y;
                    }
                    if constexpr (PAIRS % 2)
                        xw[i][PAIRS - 1] =
                            *reinterpret_cast<const uint64_t *>(wptr + i * row_bytes + 8 * (PAIRS - 1));
                }
                // one walk over the stage's channels: taps, "next channel" (window reload), end
                if constexpr (R == 4 && PT == 4 && PS == 8) {
                    SPC2_DISPATCH_R4T4S8(acc, xw, sp, wp, ch_bytes, row_bytes);
                } else if constexpr (R == 2 && PT == 8 && PS == 4) {
                    SPC2_DISPATCH_R2T8S4(acc, xw, sp, wp, ch_bytes, row_bytes);
                } else if constexpr (R == 4 && PT == 7 && PS == 4) {
                    SPC2_DISPATCH_R4T7S4(acc, xw, sp, wp, ch_bytes, row_bytes);
                } else if constexpr (R == 2 && PT == 7 && PS == 4) {
                    SPC2_DISPATCH_R2T7S4(acc, xw, sp, wp, ch_bytes, row_bytes);
                } else {
                    static_assert(R == 4 && PT == 8 && PS == 4, "no dispatcher generated for this variant");
                    SPC2_DISPATCH_R4T8S4(acc, xw, sp, wp, ch_bytes, row_bytes);
                }
                }
                } // cl0 < cl1
            }
            SPC_PROF_MARK(3);
            // release stage s: the last warp to finish with it refills it with stage kk + ns.
            // Every warp arrives on the stage's "empty" mbarrier (release); a shared
            // counter picks the last arriver, which waits on that barrier phase
            // (acquire: all warps' reads of the stage happen before) and then orders
            // the generic-proxy reads before its async-proxy writes (fill_stage).
            __syncwarp();
            int last = 0;
            if (lane == 0) {
                mbar_arrive(smem_u32(&empty_bar[s]));
                // monotonic: the n-th use of stage s completes when the count reaches n*nwarps
                const int old = atomicAdd(&done_cnt[s], 1);
                last = old == rnd * nwarps + nwarps - 1;
                if (last) mbar_wait(smem_u32(&empty_bar[s]), rnd & 1);
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last && kk + ns < total) {
                if (STG == 0 || lane == 0) fill(kk + ns, s); // (kk + ns) % ns == s
            }
            SPC_PROF_MARK(0);
            ++kk;
            if (++s == ns) {
                s = 0;
                ++rnd;
            }
        }
        SPC_PROF_MARK(4);
        if (!active) continue;
        if (kind == 1) {
            SPC_PROF_MARK(5);
            // park: the partial sums go to slot (b, warp) for CTA b+1
            const size_t slot = size_t(bid) * a.gpc + warp;
            ulonglong2 *dst = a.sk_part + slot * (R * PT * SH / 2) * 32 + lane;
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int t = 0; t < PT; ++t)
#pragma unroll
                    for (int h = 0; h < SH; h += 2)
                        __stcg(dst + size_t(((r * PT + t) * SH + h) / 2) * 32, make_ulonglong2(acc[r][t][h], acc[r][t][h + 1]));
            __threadfence();
            __syncwarp();
            if (lane == 0)
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.sk_flag + slot), "l"(a.epoch) : "memory");
            if (tr && threadIdx.x == 0) tr[1] = gtimer();
            SPC_PROF_MARK(4);
            continue;
        }

        // ---------------- epilogue (a6) ----------------
        int n = un.n0 + im, ty = un.ty0 + tyl;
        if (a.band) {
            const int v = un.n0 + im;
            n = v / a.tiles_y;
            ty = v - n * a.tiles_y;
        }
        // (a column block's extra lane computes the next block's first tile: not stored)
        const bool own = !CB || tx < a.cb_tiles;
        const bool out_ok = lane_ok && own && n < a.N && ty < a.tiles_y;
        const int oy0 = ty * PT, ox0 = ((CB ? un.cb * a.cb_tiles : 0) + tx) * PS - XS;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int f = s_rows[g * R + r];
        if (f < 0) continue; // warp-uniform
        const float b = s_bias[f];
        float v[PT][PS];
#pragma unroll
        for (int t = 0; t < PT; ++t)
#pragma unroll
            for (int h = 0; h < SH; ++h) {
                v[t][2 * h] = __fadd_rn(lo_f(acc[r][t][h]), b);
                v[t][2 * h + 1] = __fadd_rn(hi_f(acc[r][t][h]), b);
            }
        if constexpr (!FUSED) {
            if (!out_ok) continue;
            const size_t plane = ((size_t)n * a.F + f) * a.Ho * a.Wo;
            float *yp = a.y + plane;
#pragma unroll
            for (int t = 0; t < PT; ++t) {
                const int oy = oy0 + t;
                if (oy >= a.Ho) continue;
                float *row = yp + (size_t)oy * a.Wo;
                const float *rrow = (EPI & 2) ? a.res + plane + (size_t)oy * a.Wo : nullptr;
                if (XS == 0 && ox0 + PS <= a.Wo && ((reinterpret_cast<uintptr_t>(row + ox0) & 15) == 0) &&
                    (a.Wo & 3) == 0 && (!(EPI & 2) || ((reinterpret_cast<uintptr_t>(rrow + ox0) & 15) == 0))) {
#pragma unroll
                    for (int q = 0; q < PS; q += 4) {
                        float4 o = make_float4(v[t][q], v[t][q + 1], v[t][q + 2], v[t][q + 3]);
                        if constexpr ((EPI & 2) != 0) {
                            const float4 rr = *reinterpret_cast<const float4 *>(rrow + ox0 + q);
                            o.x = __fadd_rn(o.x, rr.x); o.y = __fadd_rn(o.y, rr.y);
                            o.z = __fadd_rn(o.z, rr.z); o.w = __fadd_rn(o.w, rr.w);
                        }
                        if constexpr ((EPI & 1) != 0) {
                            o.x = o.x > 0.0f ? o.x : 0.0f; o.y = o.y > 0.0f ? o.y : 0.0f;
                            o.z = o.z > 0.0f ? o.z : 0.0f; o.w = o.w > 0.0f ? o.w : 0.0f;
                        }
                        *reinterpret_cast<float4 *>(row + ox0 + q) = o;
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < PS; ++q) {
                        const int ox = ox0 + q;
                        if (ox >= 0 && ox < a.Wo) {
                            float o = v[t][q];
                            if constexpr ((EPI & 2) != 0) o = __fadd_rn(o, rrow[ox]);
                            if constexpr ((EPI & 1) != 0) o = o > 0.0f ? o : 0.0f;
                            row[ox] = o;
                        }
                    }
                }
            }
        } else {
            // ReLU then 2x2 max with first-max argmax (row-major window order).
            // XS == 0: the pairs (0,1), (2,3), ... of the tile are lane-local.  XS == 3:
            // the tile covers columns PS*tx-3 .. PS*tx+PS-4; pairs (1,2), (3,4), ... are
            // local and the last pair (PS-1, PS) takes column PS*tx+PS-3 from the next
            // lane (the pair (-1, 0) is the previous lane's).  A lane whose neighbour
            // is another tile row never needs it: its last pair starts at >= Wo - 1.
            float rl[PT][PS + 1];
#pragma unroll
            for (int t = 0; t < PT; ++t) {
#pragma unroll
                for (int q = 0; q < PS; ++q) rl[t][q] = v[t][q] > 0.0f ? v[t][q] : 0.0f;
                rl[t][PS] = XS ? __shfl_down_sync(0xffffffffu, rl[t][0], 1) : 0.0f;
            }
            if (!out_ok) continue;
            float *yp = a.y + ((size_t)n * a.F + f) * a.Po * a.Qo;
            int32_t *ap = a.argmax ? a.argmax + ((size_t)n * a.F + f) * a.Po * a.Qo : nullptr;
#pragma unroll
            for (int tp = 0; tp < PT / 2; ++tp) {
                const int py = (oy0 >> 1) + tp;
                if (py >= a.Po) continue;
#pragma unroll
                for (int pp = 0; pp < PS / 2; ++pp) {
                    const int q0 = XS ? 2 * pp + 1 : 2 * pp;
                    const int ox = ox0 + q0;
                    if (ox < 0) continue;
                    const int px = ox >> 1;
                    if (px >= a.Qo) continue;
                    float best = 0.0f;
                    int bidx = 0;
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const int dy = w >> 1, dx = w & 1;
                        const float rv = rl[2 * tp + dy][q0 + dx];
                        if (w == 0 || rv > best) {
                            best = rv;
                            bidx = (oy0 + 2 * tp + dy) * a.Wo + ox + dx;
                        }
                    }
                    yp[(size_t)py * a.Qo + px] = best;
                    if (ap) ap[(size_t)py * a.Qo + px] = bidx;
                }
            }
        }
    }
    }
    SPC_PROF_MARK(7);
    if (a.sk) {
        // the last CTA to finish resets the arrival counters for the next launch on
        // this workspace (every CTA has taken its ticket by then)
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
    SPC_PROF_MARK(0);
#ifdef SPC_PROF
    __syncthreads();
    if (a.prof && threadIdx.x < 9) atomicAdd(a.prof + threadIdx.x, s_prof[threadIdx.x]);
#endif
    if (tr && threadIdx.x == 0) tr[2] = gtimer();
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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


template <int R, int PT, int PS, bool FUSED, int XS, int DISP, int STG, int EPI = 0>
cudaError_t launch_one(const CUtensorMap &map, const PipeArgs &a, int grid, size_t smem, cudaStream_t s,
                       bool pdl) {
    auto kern = pipe_kernel<R, PT, PS, FUSED, XS, DISP, STG, EPI>;
    static size_t attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    size_t &done = attr_done[dev & 63];
    if (smem > 48 * 1024 && __atomic_load_n(&done, __ATOMIC_ACQUIRE) < smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        __atomic_store_n(&done, smem, __ATOMIC_RELEASE);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(unsigned(32 * a.gpc));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, map, a);
}

// Shared-memory wavefronts of one warp-wide window row load (LDS.128 at the
// window start + LDS.64 at +16 B) for a candidate pitch: quarter-warp phases
// for 16-byte accesses, half-warp phases for 8-byte accesses; the degree of a
// phase is the largest number of distinct addresses that share a bank.
int window_wavefronts(const PipeGeometry &g, int pitch) {
    const int PT = g.T, PS = g.S;
    int addr[32];
    for (int l = 0; l < 32; ++l) {
        const int li = l < g.lanes ? l : 0;
        int im, tyl, tx;
        lane_tile(li, g.lane_order, g.ipb, g.tr, g.tiles_x, im, tyl, tx);
        addr[l] = (im * g.cc * g.rs + tyl * PT) * pitch + tx * PS; // words (slot im of the stage)
    }
    int total = 0;
    for (int pass = 0; pass < 2; ++pass) {
        const int width = pass == 0 ? 4 : 2, group = pass == 0 ? 8 : 16, off = pass == 0 ? 0 : PS;
        for (int p0 = 0; p0 < 32; p0 += group) {
            int worst = 1;
            for (int bank = 0; bank < 32; ++bank) {
                int distinct[32], nd = 0;
                for (int l = p0; l < p0 + group; ++l) {
                    for (int w = 0; w < width; ++w) {
                        const int word = addr[l] + off + w;
                        if ((word & 31) != bank) continue;
                        bool seen = false;
                        for (int d = 0; d < nd; ++d) seen |= distinct[d] == word;
                        if (!seen) distinct[nd++] = word;
                    }
                }
                worst = std::max(worst, nd);
            }
            total += worst;
        }
    }
    return total;
}

} // namespace

void read_pipe_knobs(PipeKnobs &k) {
    k = PipeKnobs{};
    if (const char *e = std::getenv("SPCONV_PIPE_STAGING")) {
        if (std::strcmp(e, "cp") == 0) k.staging = 2;
        if (std::strcmp(e, "pad") == 0) k.staging = 1;
    }
    if (const char *e = std::getenv("SPCONV_PIPE_SK")) k.sk = e[0] == '1' ? 1 : 0;
    if (const char *e = std::getenv("SPCONV_PIPE_REV")) k.rev = e[0] == '1';
    if (const char *e = std::getenv("SPCONV_PIPE_SK_SPLIT")) k.sk_split = !(std::strcmp(e, "uniform") == 0 || e[0] == '0');
    if (const char *e = std::getenv("SPCONV_PDL")) k.pdl = !(e[0] == '0');
    if (const char *e = std::getenv("SPCONV_PIPE_TRACE")) std::snprintf(k.trace, sizeof(k.trace), "%s", e);
    if (const char *e = std::getenv("SPCONV_PIPE_PROF")) std::snprintf(k.prof, sizeof(k.prof), "%s", e);
    if (const char *e = std::getenv("SPCONV_DEBUG")) k.debug = e[0] == '1';
    if (const char *e = std::getenv("SPCONV_DENSE_STAGE_BYTES")) k.dense_stage = std::max(4096, std::atoi(e));
}

bool pipe_supported(int C, int H, int W, int F, int K, int stride, int pad) {
    (void)C; (void)F; (void)H;
    // 32-pixel (8x4) tiles; rows wider than 32 tiles (Wo + 3 > 128) are split into
    // column blocks (pipe_geometry).  Inputs whose rows TMA cannot stage directly
    // (W % 4 != 0 or a misaligned base) go through a left-padded copy (launch_pipe).
    return K == 3 && stride == 1 && pad == 1 && W <= 8192;
}

void pipe_geometry(const Plan &p, int mode, PipeGeometry &g, int T) {
    // mode 0: TMA on the caller's tensor (xs = 3); 1: TMA on the left-padded copy
    // (xs = 0); 2: cp.async staging (xs = 0)
    g = PipeGeometry{};
    const bool tma = mode != 2;
    g.xs = mode == 0 ? 3 : 0;
    // 32-pixel thread tiles: 16 FFMA2 per nonzero (scripts/probes/dispatch_probe.cu).
    // 8x4 (tall) keeps the window's 128-bit loads at a 16-byte lane stride (fewer bank
    // conflicts than 4x8, measured 11.3 vs 9.5 TFLOP/s on c2).  T = 7 (7x4 tiles) serves
    // conv-only calls on images whose height is a multiple of 7 but not of 8 (c4's 14x14,
    // VGG's 28x28): 100% instead of 87.5% row coverage.
    g.T = T;
    g.S = 4;
    const int PT = g.T, PS = g.S;
    g.tiles_x = (p.Wo + g.xs + PS - 1) / PS;
    g.tiles_y = (p.Ho + PT - 1) / PT;
    g.tiles_total = g.tiles_x;
    g.colblocks = 1;
    g.cb_tiles = g.tiles_x;
    if (g.tiles_x > 32) {
        // wide rows (Wo > 125): column blocks of cb_tiles tiles, each staged with its own
        // halo; the lanes of a block cover one extra tile (its pool-pair neighbour)
        g.colblocks = (g.tiles_x + 30) / 31;
        g.cb_tiles = (g.tiles_x + g.colblocks - 1) / g.colblocks;
        g.tiles_x = g.cb_tiles + 1; // lanes per tile row
    }
    const int per_img = g.tiles_x * g.tiles_y;
    if (per_img <= 16) {
        g.ipb = 32 / per_img;
        g.tr = g.tiles_y;
    } else {
        g.ipb = 1;
        g.tr = std::min(g.tiles_y, 32 / g.tiles_x);
    }
    // band mode: when whole-image blocks of tr tile rows leave a ragged last block
    // (c2: 7 tile rows in blocks of 2), a unit takes tr bands of ONE tile row each
    // from the flattened (image, tile row) sequence instead, each staged with its
    // own halo -- no half-empty units (SPCONV_PIPE_BANDS=0 disables)
    g.band = 0;
    if (g.ipb == 1 && g.tr > 1 && g.tiles_y % g.tr != 0) {
        const char *e = std::getenv("SPCONV_PIPE_BANDS");
        if (!(e && e[0] == '0')) {
            g.band = 1;
            g.ipb = g.tr;
            g.tr = 1;
        }
    }
    g.lanes = g.ipb * g.tr * g.tiles_x;
    g.blocks_y = g.band ? 1 : (g.tiles_y + g.tr - 1) / g.tr;
    g.rs = PT * g.tr + 2;
    g.cc = p.pipe_cc;
    // smem columns read: window of the last tile ends at 4*(tiles_x-1) + 5
    const int need = ((PS * g.tiles_x + 2) + 3) & ~3;
    int best = need, best_wf = 1 << 30, best_order = 0, best_rs = g.rs;
    // the lane order matters only with several images AND several tile rows per unit
    // (c4: 4 images x 2 tile rows: the pitch alone cannot separate the quarter-warp's
    // two tile rows, 8*pitch = 0 mod 32 words; the image slots can be: 12 -> 8
    // wavefronts per window row).  The slots' row count may also be padded by up to 3
    // rows (staged but unused) when that separates them (c4 with 7-row tiles: 16 rows
    // per slot put every slot on the same banks, 18 do not); band slots are not padded
    // (a band's start row is derived from rs).
    const int orders = (g.ipb > 1 && g.tr > 1) ? 2 : 1;
    const int rs0 = g.rs, extra_rows = (g.band || g.ipb == 1) ? 0 : 3;
    for (int extra = 0; extra <= extra_rows; ++extra) {
        g.rs = rs0 + extra;
        for (int order = 0; order < orders; ++order) {
            g.lane_order = order;
            for (int cand = need; cand <= need + 32; cand += 4) {
                // band mode stages every band with its own TMA box into slot b of the stage:
                // slots must start on 128-byte boundaries (the tensor-copy destination
                // alignment), i.e. cc * rs * pitch words must be a multiple of 32 (a pitch
                // multiple of 16 words always qualifies, and the range holds two)
                if (g.band && (g.cc * g.rs * cand) % 32 != 0) continue;
                const int wf = window_wavefronts(g, cand);
                // fewest wavefronts; among equals the smallest staged box
                if (wf < best_wf || (wf == best_wf && g.rs * cand < best_rs * best)) {
                    best_wf = wf;
                    best = cand;
                    best_order = order;
                    best_rs = g.rs;
                }
            }
        }
    }
    g.pitch = best;
    g.lane_order = best_order;
    g.rs = best_rs;
    if (g.band && (g.cc * g.rs * g.pitch) % 32 != 0) return; // (unreachable: see the search)
    if (tma && (g.pitch > 256 || g.rs > 256)) return;
    if (mode == 0 && (p.W * 4) % 16 != 0) return;
    g.nchunks = (p.C + g.cc - 1) / g.cc;
    g.in_words = g.ipb * g.cc * g.rs * g.pitch;
    g.in_pad = (g.in_words * 4 + 127) & ~127;
    g.st_bytes = (p.max_chunk_bytes + 32 + 127) & ~127; // + 2 entries of look-ahead slack
    const int stage_bytes = g.in_pad + g.st_bytes;
    const int cstart_bytes = ((p.num_gsets * (g.nchunks + 1) + p.num_groups * p.R + p.F) * 4 + 15) & ~15;
    const int budget = 220 * 1024 - cstart_bytes;
    g.nstage = std::min(MAXSTAGE, budget / stage_bytes);
    if (g.nstage < 2) return;
    g.smem_bytes = size_t(g.nstage) * stage_bytes + cstart_bytes;
    g.ok = true;
}

// Left-padded copy for inputs TMA cannot stage directly (row stride not a
// multiple of 16 bytes, or a misaligned base): xp[n][c][iy][0] = 0,
// xp[..][1 + ix] = x[..][ix], zero up to the padded width Wp (multiple of 4).
__global__ void __launch_bounds__(256) pad_rows_kernel(const float *__restrict__ x, float *__restrict__ xp,
                                                       int64_t rows, int W, int Wp) {
    const int q = Wp / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * q;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / q;
        const int c0 = int(i - row * q) * 4;
        const float *src = x + row * W;
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int ix = c0 + k - 1;
            v[k] = (ix >= 0 && ix < W) ? __ldg(src + ix) : 0.0f;
        }
        reinterpret_cast<float4 *>(xp + row * Wp)[c0 / 4] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

void keep_pool_cached() {
    // Workspaces come from the device's default stream-ordered pool; keep freed
    // blocks cached in it (release threshold = max) so a steady stream of calls
    // does not return memory to the driver at every synchronisation.
    static bool pool_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!pool_set[dev & 63]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
        pool_set[dev & 63] = true;
    }
}

int sm_count_of_current_device() {
    static int sm_count[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!sm_count[dev & 63]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        sm_count[dev & 63] = v;
    }
    return sm_count[dev & 63];
}

unsigned long long next_sk_epoch() {
    // a tagged, process-unique value: stale workspace contents never equal it
    static std::atomic<unsigned long long> epochs{0};
    return 0x5ec0'0000'0000'0000ull | (++epochs & 0x0000'ffff'ffff'ffffull);
}

cudaError_t SkWorkspace::release(cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    if (async && base) e = cudaFreeAsync(base, s);
    base = nullptr;
    if (lock.owns_lock()) lock.unlock();
    return e;
}

// The stream-K workspace of a launch on stream s (pipe and dense kernels): layout
// [0, 512) 64 counter slots {arrival ticket, finished CTAs} (0 when unused), [512, ...)
// one u64 flag per (CTA, warp), parked partial sums from kSkHeader on.  Launch k on a
// workspace uses counter slot k % 64 -- consecutive launches on a stream (which overlap
// under programmatic dependent launch) never share a slot, and each launch's last CTA
// to finish zeroes its slot -- so a CTA can take its ticket BEFORE griddepcontrol.wait.
// One workspace per (plan, stream), kept and grown; the plan's workspace lock is HELD
// in w until w.release(), so a concurrent call on the same stream cannot replace the
// buffer between this lookup and its launch.  Under stream capture, or beyond 8
// streams, a stream-ordered (zeroed) allocation per call.
cudaError_t stream_k_workspace(const Plan &p, cudaStream_t s, size_t part_bytes, int nflags, SkWorkspace &w) {
    const size_t need = kSkHeader + part_bytes;
    if (kSkFlags + size_t(nflags) * 8 > kSkHeader) return cudaErrorInvalidConfiguration;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    bool cached = cap == cudaStreamCaptureStatusNone;
    Plan &mp = const_cast<Plan &>(p);
    if (cached) {
        w.lock = std::unique_lock<std::mutex>(mp.sk_mu);
        bool known = false;
        for (auto &x : mp.sk_ws) known |= x.stream == s;
        cached = known || mp.sk_ws.size() < 8;
        if (!cached) w.lock.unlock();
    }
    unsigned slot = 0;
    if (!cached) {
        keep_pool_cached();
        cudaError_t e = cudaMallocAsync(&w.base, need, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(w.base, 0, kSkHeader, s);
        if (e != cudaSuccess) {
            if (w.base) cudaFreeAsync(w.base, s);
            w.base = nullptr;
            return e;
        }
        w.async = true;
    } else {
        Plan::SkSlot *ws = nullptr;
        for (auto &x : mp.sk_ws)
            if (x.stream == s) ws = &x;
        if (!ws) {
            mp.sk_ws.push_back(Plan::SkSlot{s, nullptr, 0, 0});
            ws = &mp.sk_ws.back();
        }
        if (ws->bytes < need) {
            if (ws->ptr) {
                // the old buffer may still be in use by earlier launches on s
                cudaStreamSynchronize(s);
                cudaFree(ws->ptr);
                ws->ptr = nullptr;
                ws->bytes = 0;
            }
            cudaError_t e = cudaMalloc(&ws->ptr, need);
            if (e != cudaSuccess) return e;
            ws->bytes = need;
            ws->seq = 0;
            cudaMemsetAsync(ws->ptr, 0, kSkHeader, s); // counters and flags start at 0
        }
        w.base = ws->ptr;
        slot = ws->seq++ % unsigned(kSkSlots);
    }
    char *b = static_cast<char *>(w.base);
    w.ticket = reinterpret_cast<unsigned *>(b) + 2 * slot;
    w.flag = reinterpret_cast<unsigned long long *>(b + kSkFlags);
    w.part = b + kSkHeader;
    return cudaSuccess;
}

// The launch schedule of one forward of N images (staging mode, units, persistent
// grid, stream-K): the single source of these decisions for launch_pipe and for the
// spconv_launch_info query the tests assert on.
bool pipe_schedule(const Plan &p, int N, uintptr_t x, PipeSchedule &q, bool conv_only, int epi) {
    q = PipeSchedule{};
    // staging: 0 = TMA on the caller's tensor (tile columns shifted by 3),
    //          1 = TMA on a left-padded copy (no shift), 2 = cp.async (fallback)
    const bool x16 = (x & 15) == 0;
    int mode = (p.pipe_tma.ok && x16) ? 0 : p.pipe_pad.ok ? 1 : 2;
    if (p.knobs.staging == 2) mode = 2;
    if (p.knobs.staging == 1 && p.pipe_pad.ok) mode = 1;
    if (mode != 2 && get_encode() == nullptr) mode = 2;
    const PipeGeometry *gp = mode == 0 ? &p.pipe_tma : mode == 1 ? &p.pipe_pad : &p.pipe_cp;
    // non-fused calls take the 7-row-tile geometry when the plan has one (TMA modes)
    if (conv_only && p.pipe_dispatch == 0 && mode != 2) {
        const PipeGeometry &g7 = mode == 0 ? p.pipe7_tma : p.pipe7_pad;
        if (g7.ok) gp = &g7;
    }
    const PipeGeometry &g = *gp;
    if (!g.ok) return false;
    // wide rows (column blocks) are instantiated for TMA staging with the plain
    // epilogue and the default dispatcher only (launch_pipe)
    if (g.colblocks > 1 && (mode == 2 || epi != 0 || p.pipe_dispatch != 0)) return false;
    q.mode = mode;
    q.g = &g;
    const int64_t nblocks = g.band ? (int64_t(N) * g.tiles_y + g.ipb - 1) / g.ipb
                                   : (int64_t)((N + g.ipb - 1) / g.ipb) * g.blocks_y;
    q.nunits = nblocks * g.colblocks * p.num_gsets;
    if (q.nunits > 0x7fffffff) return false;
    // persistent: one CTA per SM (the register file holds one 8-warp CTA)
    q.grid = int(std::min<int64_t>(q.nunits, sm_count_of_current_device()));
    // ordered stream-K when the units do not divide evenly over the persistent CTAs
    // and the last partial round is a noticeable share of the work (c2: 224 units on
    // 148 SMs = 1.51 rounds -> 2 without it)
    q.sk = q.nunits > q.grid && q.nunits % q.grid != 0 && q.nunits < 16 * int64_t(q.grid);
    if (p.knobs.sk >= 0) q.sk = p.knobs.sk == 1 && q.nunits > q.grid;
    q.launches = mode == 1 ? 2 : 1;
    return true;
}

// Per-warp stream-K split points.  The uniform split gives every CTA the same number
// of (unit, channel) steps, but a warp's time is its own group's walk: its taps and
// window reloads in those channels, which differ between the warps of a CTA (measured
// on c2: the average warp waits 5% of the kernel at the end for its CTA's slowest) and
// between CTAs, plus per-item costs (a unit epilogue, a park, a resume; CTAs with an
// extra whole unit ended ~3 us later).  Here (1) the CTA boundaries B_b are placed so
// that every CTA's range costs the same T (greedy + bisection on T) in the average
// warp's walk cost + item costs, and (2) inside the unit of B_b each warp w splits at
// the channel where ITS cumulative cost reaches its share of the boundary's cumulative
// cost -- so every warp of every CTA walks the same cost.  Only split points move: every
// output is still one ascending fma chain (the ordered head/tail hand-off per warp).
void sk_split_core(const float *lane_cost, int C, int gpc, int ngs, int num_groups, int cc, int64_t U, int G, bool fused,
                   std::vector<int32_t> &unit_out, std::vector<uint16_t> &ch_out) {
    const double kEpi = fused ? kSkEpiFused : kSkEpiConv;
    // per (gset, lane) prefix costs over the channels, and per gset the lane average
    std::vector<double> pre(size_t(ngs) * gpc * (C + 1), 0.0), apre(size_t(ngs) * (C + 1), 0.0);
    std::vector<double> wtot(size_t(gpc), 0.0); // per lane: cost of one unit of every gset
    double atot = 0.0;
    for (int gs = 0; gs < ngs; ++gs) {
        // a unit takes about one warp's walk whatever the number of active warps (the
        // walk is latency bound): the CTA-level cost averages the ACTIVE lanes only
        const int act = std::max(1, std::min(gpc, num_groups - gs * gpc));
        for (int w = 0; w < gpc; ++w) {
            double *P = &pre[(size_t(gs) * gpc + w) * (C + 1)];
            for (int c = 0; c < C; ++c) P[c + 1] = P[c] + lane_cost[(size_t(gs) * gpc + w) * C + c];
            if (w < act)
                for (int c = 0; c <= C; ++c) apre[size_t(gs) * (C + 1) + c] += P[c] / act;
            wtot[size_t(w)] += P[C];
        }
    }
    for (int gs = 0; gs < ngs; ++gs) atot += apre[size_t(gs) * (C + 1) + C];
    // cumulative cost at step (u, c): whole units before u (gsets cycle) + the prefix in u
    std::vector<double> agstot(static_cast<size_t>(ngs), 0.0), agcum(static_cast<size_t>(ngs) + 1, 0.0);
    for (int gs = 0; gs < ngs; ++gs) {
        agstot[size_t(gs)] = apre[size_t(gs) * (C + 1) + C];
        agcum[size_t(gs) + 1] = agcum[size_t(gs)] + agstot[size_t(gs)];
    }
    auto Fa = [&](int64_t step) {
        const int64_t u = step / C;
        const int c = int(step - u * C), gs = int(u % ngs);
        return double(u / ngs) * atot + agcum[size_t(gs)] + (c ? apre[size_t(gs) * (C + 1) + c] : 0.0);
    };
    std::vector<double> wcum(size_t(gpc) * (ngs + 1), 0.0); // per lane: units of gsets [0, gs)
    for (int w = 0; w < gpc; ++w)
        for (int gs = 0; gs < ngs; ++gs)
            wcum[size_t(w) * (ngs + 1) + gs + 1] =
                wcum[size_t(w) * (ngs + 1) + gs] + pre[(size_t(gs) * gpc + w) * (C + 1) + C];
    auto Fw = [&](int w, int64_t step) {
        const int64_t u = step / C;
        const int c = int(step - u * C), gs0 = int(u % ngs);
        return double(u / ngs) * wtot[size_t(w)] + wcum[size_t(w) * (ngs + 1) + gs0] +
               pre[(size_t(gs0) * gpc + w) * (C + 1) + c];
    };
    const int64_t total = U * C;
    auto cost = [&](int64_t s0, int64_t e0) {
        double v = Fa(e0) - Fa(s0);
        if (s0 % C) v += kSkResume;
        v += kEpi * double(e0 / C - s0 / C); // units finished in (s0, e0]
        if (e0 % C) v += kSkPark;
        return v;
    };
    // CTA boundaries: CTA b takes the remaining cost / remaining CTAs (each further
    // split adds a park and a resume), the boundary nearest to that share
    std::vector<int64_t> B(size_t(G) + 1, 0);
    int64_t s0 = 0;
    for (int b = 0; b < G - 1; ++b) {
        B[size_t(b)] = s0;
        if (s0 >= total) continue;
        const double share = (cost(s0, total) + double(G - b - 1) * (kSkPark + kSkResume)) / double(G - b);
        const int64_t emin = (s0 % C) ? (s0 / C + 1) * C : s0 + 1; // a tail finishes its unit
        int64_t lo = std::min(emin, total), hi = total;
        if (cost(s0, lo) <= share) {
            while (lo < hi) { // largest e with cost(s0, e) <= share
                const int64_t mid = lo + (hi - lo + 1) / 2;
                if (cost(s0, mid) <= share) lo = mid; else hi = mid - 1;
            }
            if (lo < total && cost(s0, lo + 1) - share < share - cost(s0, lo)) ++lo; // nearest
        }
        s0 = lo;
    }
    B[size_t(G) - 1] = s0;
    B[size_t(G)] = total;
    unit_out.assign(size_t(G) + 1, 0);
    ch_out.assign((size_t(G) + 1) * gpc, 0);
    unit_out[size_t(G)] = int32_t(U);
    for (int b = 1; b < G; ++b) {
        const int64_t s0 = B[size_t(b)];
        int64_t u = s0 / C;
        uint16_t *row = &ch_out[size_t(b) * gpc];
        if (s0 % C) {
            // each lane splits where its own cumulative cost reaches its share, at most
            // one stage from the CTA-level split: the head and tail stage ranges are
            // the union over the lanes, and a lane whose group costs differ much from
            // the average (R = 2 on c4: 11 group sets, a ragged one) would otherwise
            // stretch both over the whole unit (measured: c4_50 291 -> 406 us)
            const double target = Fa(s0) / Fa(total);
            const int h = int(s0 % C), clo = std::max(0, h - cc), chi = std::min(C, h + cc);
            int mx = 0, mn = C;
            const int gsu = int(u % ngs);
            for (int w = 0; w < gpc; ++w) {
                if (gsu * gpc + w >= num_groups) continue; // no group in this unit: set below
                const double tw = target * Fw(w, total);
                int c = clo; // (the result is clamped to [clo, chi] anyway)
                while (c < chi && Fw(w, u * C + c + 1) <= tw) ++c;
                if (c < chi && Fw(w, u * C + c + 1) - tw < tw - Fw(w, u * C + c)) ++c; // nearest
                row[w] = uint16_t(c);
                mx = std::max(mx, c);
                mn = std::min(mn, c);
            }
            for (int w = 0; w < gpc; ++w) // idle lanes: inside the active lanes' range
                if (gsu * gpc + w >= num_groups) row[w] = uint16_t(mx);
            if (mx == 0) { /* every lane at the unit start: no split */ }
            else if (mn == C) { // every lane at the unit end: boundary at the next unit
                ++u;
                for (int w = 0; w < gpc; ++w) row[w] = 0;
            }
        }
        unit_out[size_t(b)] = int32_t(u);
    }
    // ranges must stay ordered and cover at least one unit boundary each (no middle
    // pieces); otherwise fall back to the uniform split
    bool ok = true;
    for (int b = 0; b < G && ok; ++b) {
        const int u0 = unit_out[size_t(b)], u1 = unit_out[size_t(b) + 1];
        int mx0 = 0, mx1 = 0;
        for (int w = 0; w < gpc; ++w) {
            mx0 = std::max(mx0, int(ch_out[size_t(b) * gpc + w]));
            mx1 = std::max(mx1, int(ch_out[(size_t(b) + 1) * gpc + w]));
        }
        if (u1 < u0 || (mx0 > 0 && u1 <= u0)) ok = false; // (u1 == u0 without a tail: head only)
    }
    if (!ok) unit_out.clear();
}

void sk_split(const Plan &p, int64_t U, int G, bool fused, Plan::SkTable &t) {
    sk_split_core(p.sk_cost.data(), p.C, p.gpc, p.num_gsets, p.num_groups, p.pipe_cc, U, G, fused, t.unit, t.ch);
}

// The per-warp split table of a stream-K launch, computed once per launch shape (cached
// in the plan): copied to unit / ch (kernel-parameter layout) when given; false = the
// uniform split (knob off, grid or warps beyond the parameter table, no valid split).
bool sk_table(const Plan &p, const PipeSchedule &q, int N, bool fused, int32_t *unit, uint16_t *ch) {
    if (!q.sk || !p.knobs.sk_split || q.grid > kSkTabCta || p.gpc > kSkTabGpc || p.sk_cost.empty()) return false;
    Plan &mp = const_cast<Plan &>(p);
    std::lock_guard<std::mutex> lk(mp.cache.mu);
    Plan::SkTable *t = nullptr;
    for (auto &e : mp.sk_tab)
        if (e.N == N && e.grid == q.grid && e.fused == int(fused) && e.geo == q.g) t = &e;
    if (!t) {
        t = &mp.sk_tab[mp.sk_tab_next];
        mp.sk_tab_next = (mp.sk_tab_next + 1) % 4;
        *t = Plan::SkTable{};
        sk_split(p, q.nunits, q.grid, fused, *t);
        t->N = N; t->grid = q.grid; t->fused = int(fused); t->geo = q.g;
    }
    if (t->unit.empty()) return false;
    if (unit)
        for (int b = 0; b <= q.grid; ++b) {
            unit[b] = t->unit[size_t(b)];
            for (int w = 0; w < p.gpc; ++w) ch[b * kSkTabGpc + w] = t->ch[size_t(b) * p.gpc + w];
        }
    return true;
}

cudaError_t launch_pipe(const Plan &p, int N, const float *x, float *y, int32_t *argmax, bool fused,
                        cudaStream_t s, const float *res, int epi) {
    PipeSchedule sched;
    if (!pipe_schedule(p, N, reinterpret_cast<uintptr_t>(x), sched, !fused, epi))
        return cudaErrorInvalidConfiguration;
    const int mode = sched.mode;
    const PipeGeometry &g = *sched.g;
    const int Wp = ((p.W + 2) + 3) & ~3;
    float *xp = nullptr;
    if (mode == 1) {
        const size_t bytes = size_t(N) * p.C * p.H * Wp * 4;
        keep_pool_cached();
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&xp), bytes, s);
        if (e != cudaSuccess) return e;
        const int64_t rows = int64_t(N) * p.C * p.H;
        const int64_t work = rows * (Wp / 4);
        const int blocks = int(std::min<int64_t>((work + 255) / 256, 148 * 16));
        pad_rows_kernel<<<blocks, 256, 0, s>>>(x, xp, rows, p.W, Wp);
        if ((e = cudaGetLastError()) != cudaSuccess) {
            cudaFreeAsync(xp, s);
            return e;
        }
    }
    PipeArgs a;
    a.x = x; a.y = y; a.argmax = argmax; a.res = res;
    a.bias = p.d_bias; a.group_rows = p.d_group_rows; a.chunk_start = p.d_chunk_start;
    a.stream = reinterpret_cast<const char *>(p.d_stream2);
    a.N = N; a.C = p.C; a.H = p.H; a.W = p.W; a.F = p.F; a.Ho = p.Ho; a.Wo = p.Wo;
    a.Po = p.Ho / 2; a.Qo = p.Wo / 2;
    a.xs = g.xs; a.tiles_x = g.tiles_x; a.tiles_y = g.tiles_y; a.ipb = g.ipb; a.tr = g.tr;
    a.colblocks = g.colblocks; a.cb_tiles = g.cb_tiles; a.tiles_total = g.tiles_total;
    a.lanes = g.lanes; a.blocks_y = g.blocks_y; a.rs = g.rs; a.pitch = g.pitch; a.nstage = g.nstage;
    a.in_words = g.in_words; a.in_pad = g.in_pad; a.st_bytes = g.st_bytes;
    a.cc = g.cc; a.nchunks = g.nchunks; a.band = g.band;
    for (int l = 0; l < 32; ++l) {
        int im, tyl, tx;
        lane_tile(l < g.lanes ? l : 0, g.lane_order, g.ipb, g.tr, g.tiles_x, im, tyl, tx);
        a.lane_map[l] = (uint32_t(im) << 16) | (uint32_t(tyl) << 8) | uint32_t(tx);
    }
    a.gpc = p.gpc; a.num_groups = p.num_groups; a.num_gsets = p.num_gsets;
    a.tma = mode != 2 ? 1 : 0;
    a.ent = 8;
    a.sk_tab = 0;
    const int64_t nunits = sched.nunits;

    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    const void *map_src = mode == 0 ? static_cast<const void *>(x) : static_cast<const void *>(xp);
    Plan &mp = const_cast<Plan &>(p);
    if (mode != 2 && !mp.cache.find_map(map_src, N, &g, map)) {
        const cuuint64_t Wt = mode == 0 ? (cuuint64_t)p.W : (cuuint64_t)Wp;
        cuuint64_t dims[4] = {Wt, (cuuint64_t)p.H, (cuuint64_t)p.C, (cuuint64_t)N};
        cuuint64_t strides[3] = {Wt * 4, (cuuint64_t)p.H * Wt * 4, (cuuint64_t)p.C * p.H * Wt * 4};
        cuuint32_t box[4] = {(cuuint32_t)g.pitch, (cuuint32_t)g.rs, (cuuint32_t)g.cc, (cuuint32_t)(g.band ? 1 : g.ipb)};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                                  mode == 0 ? const_cast<float *>(x) : xp, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            if (xp) cudaFreeAsync(xp, s);
            return cudaErrorInvalidValue;
        }
        mp.cache.put_map(map_src, N, &g, map);
    }
    const int grid = sched.grid;
    a.sk = sched.sk ? 1 : 0; a.sk_part = nullptr; a.sk_flag = nullptr; a.sk_ticket = nullptr; a.epoch = 0;
    a.trace = nullptr;
    a.rev = p.knobs.rev;
    const bool tracing = p.knobs.trace[0] != 0;
    if (tracing && cudaMalloc(&a.trace, size_t(grid) * 64) == cudaSuccess) cudaMemsetAsync(a.trace, 0, size_t(grid) * 64, s);
    a.prof = nullptr;
#ifdef SPC_PROF
    const char *prof_out = p.knobs.prof;
    if (prof_out[0] && cudaMalloc(&a.prof, 9 * sizeof(unsigned long long)) == cudaSuccess)
        cudaMemsetAsync(a.prof, 0, 9 * sizeof(unsigned long long), s);
#endif
    SkWorkspace skws;
    if (a.sk) {
        const int qn = p.R * g.T * g.S / 4;
        const size_t part_bytes = size_t(grid) * p.gpc * qn * 32 * sizeof(ulonglong2);
        cudaError_t e = stream_k_workspace(p, s, part_bytes, grid * p.gpc, skws);
        if (e != cudaSuccess) {
            if (xp) cudaFreeAsync(xp, s);
            return e;
        }
        a.sk_part = reinterpret_cast<ulonglong2 *>(skws.part);
        a.sk_flag = skws.flag;
        a.sk_ticket = skws.ticket;
        a.epoch = next_sk_epoch();
        a.sk_tab = sk_table(p, sched, N, fused, a.sk_unit, a.sk_ch) ? 1 : 0;
    }
    cudaError_t err = cudaErrorInvalidValue;
#define SPC_PIPE_MODES(RR, TT, SS, FF, DD, EE)                                                           \
    err = mode == 0 ? launch_one<RR, TT, SS, FF, 3, DD, 1, EE>(map, a, grid, g.smem_bytes, s, p.knobs.pdl != 0)              \
        : mode == 1 ? launch_one<RR, TT, SS, FF, 0, DD, 1, EE>(map, a, grid, g.smem_bytes, s, p.knobs.pdl != 0)              \
                    : launch_one<RR, TT, SS, FF, 0, DD, 0, EE>(map, a, grid, g.smem_bytes, s, p.knobs.pdl != 0);
    if (g.colblocks > 1) {
        // wide rows: TMA staging, plain epilogue, default dispatcher -- the only
        // combinations pipe_schedule accepts for them
#define SPC_PIPE_CB(RR, TT, FF)                                                                          \
    err = mode == 0 ? launch_one<RR, TT, 4, FF, 3, 0, 1, 4>(map, a, grid, g.smem_bytes, s, p.knobs.pdl != 0)  \
                    : launch_one<RR, TT, 4, FF, 0, 0, 1, 4>(map, a, grid, g.smem_bytes, s, p.knobs.pdl != 0);
        if (mode == 2 || epi != 0 || p.pipe_dispatch != 0) err = cudaErrorNotSupported;
        else if (fused && g.T == 8) {
            if (p.R == 4) { SPC_PIPE_CB(4, 8, true) } else { SPC_PIPE_CB(2, 8, true) }
        } else if (!fused && g.T == 8) {
            if (p.R == 4) { SPC_PIPE_CB(4, 8, false) } else { SPC_PIPE_CB(2, 8, false) }
        } else if (!fused && g.T == 7) {
            if (p.R == 4) { SPC_PIPE_CB(4, 7, false) } else { SPC_PIPE_CB(2, 7, false) }
        } else err = cudaErrorNotSupported;
#undef SPC_PIPE_CB
    } else if (p.R == 4 && g.T == 8 && g.S == 4) {
        if (fused) {
            if (p.pipe_dispatch == 1) { SPC_PIPE_MODES(4, 8, 4, true, 1, 0) }
            else { SPC_PIPE_MODES(4, 8, 4, true, 0, 0) }
        } else if (p.pipe_dispatch == 1) {
            if (epi != 0) err = cudaErrorNotSupported;
            else { SPC_PIPE_MODES(4, 8, 4, false, 1, 0) }
        } else if (epi == 0) { SPC_PIPE_MODES(4, 8, 4, false, 0, 0) }
        else if (epi == 1) { SPC_PIPE_MODES(4, 8, 4, false, 0, 1) }
        else if (epi == 2) { SPC_PIPE_MODES(4, 8, 4, false, 0, 2) }
        else { SPC_PIPE_MODES(4, 8, 4, false, 0, 3) }
    } else if (g.T == 7 && g.S == 4 && !fused && p.pipe_dispatch == 0 && mode != 2) {
        // 7x4 tiles: not fused (pool windows would straddle tiles), TMA staging
        // (pipe_schedule picks them only then); conv and the block epilogues
#define SPC_PIPE7(RR, EE)                                                                                  \
    err = mode == 0 ? launch_one<RR, 7, 4, false, 3, 0, 1, EE>(map, a, grid, g.smem_bytes, s, p.knobs.pdl != 0) \
                    : launch_one<RR, 7, 4, false, 0, 0, 1, EE>(map, a, grid, g.smem_bytes, s, p.knobs.pdl != 0);
        if (p.R == 4) {
            if (epi == 0) { SPC_PIPE7(4, 0) } else if (epi == 1) { SPC_PIPE7(4, 1) }
            else if (epi == 2) { SPC_PIPE7(4, 2) } else { SPC_PIPE7(4, 3) }
        } else {
            if (epi == 0) { SPC_PIPE7(2, 0) } else if (epi == 1) { SPC_PIPE7(2, 1) }
            else if (epi == 2) { SPC_PIPE7(2, 2) } else { SPC_PIPE7(2, 3) }
        }
#undef SPC_PIPE7
    } else if (p.R == 2 && g.T == 8 && g.S == 4 && p.pipe_dispatch == 0) {
        if (fused) { SPC_PIPE_MODES(2, 8, 4, true, 0, 0) }
        else if (epi == 0) { SPC_PIPE_MODES(2, 8, 4, false, 0, 0) }
        else if (epi == 1) { SPC_PIPE_MODES(2, 8, 4, false, 0, 1) }
        else if (epi == 2) { SPC_PIPE_MODES(2, 8, 4, false, 0, 2) }
        else { SPC_PIPE_MODES(2, 8, 4, false, 0, 3) }
    }
#undef SPC_PIPE_MODES
    if (a.trace) {
        // debug dump: one line per CTA (blockIdx, SM id, start, head parked, end, tail wait begin/end in ns, work index)
        std::vector<unsigned long long> h(size_t(grid) * 8);
        cudaStreamSynchronize(s);
        cudaMemcpy(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost);
        unsigned long long t0 = ~0ull;
        for (int b = 0; b < grid; ++b) t0 = std::min(t0, h[size_t(b) * 8]);
        if (FILE *f = std::fopen(p.knobs.trace, "a")) {
            for (int b = 0; b < grid; ++b) {
                const unsigned long long *e = &h[size_t(b) * 8];
                auto rel = [&](unsigned long long v) { return v ? (long long)(v - t0) : -1LL; };
                std::fprintf(f, "%d %llu %lld %lld %lld %lld %lld %llu\n", b, e[7], rel(e[0]), rel(e[1]), rel(e[2]),
                             rel(e[3]), rel(e[4]), e[5]);
            }
            std::fprintf(f, "--\n");
            std::fclose(f);
        }
        cudaFree(a.trace);
    }
#ifdef SPC_PROF
    if (a.prof) {
        // diagnostic: one line per launch: grid, warps, phase cycle sums (see the kernel)
        unsigned long long h[9];
        cudaStreamSynchronize(s);
        cudaMemcpy(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost);
        if (FILE *f = std::fopen(prof_out, "a")) {
            std::fprintf(f,
                         "grid %d warps %d other %llu wait %llu walk %llu release %llu epilogue %llu park %llu "
                         "resume %llu endsync %llu prologue %llu\n",
                         grid, grid * p.gpc, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8]);
            std::fclose(f);
        }
        cudaFree(a.prof);
    }
#endif
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
