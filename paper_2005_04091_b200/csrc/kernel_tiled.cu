// kernel_tiled.cu — register-tiled CSR sparse direct convolution for sm_100a
// (K = 3, stride 1, pad 1: the ResNet/VGG layers of BASELINE.json).
//
// What it computes is PAPER.md L393-401 (per output channel, per nonzero
// j of its CSR row: out[n][y][x] += value[j] * in[... + offset(colidx[j])]),
// with the FP32 accumulation contract of include/spconv.h (ascending colidx,
// fma, bias after the sum).  How it is laid out on B200:
//
//  * Row groups ("register blocking"):
//    output channels are partitioned into groups of R rows with balanced nnz
//    (LPT).  One warp owns one group; each lane owns a T x S output-pixel
//    tile, so a thread accumulates an R x T x S register block.
//  * Decoded stream (a2): per (group, input channel) the nonzeros of the R
//    rows as {value, id = r*9 + ky*3 + kx}, ascending id.  Within one row this
//    is ascending (ky, kx) and channels are walked in ascending order, so
//    every output still sees its row in ascending colidx order (bit-exact).
//  * Staging (a4; "array packing, data prefetching"): a CTA
//    owns 32 consecutive thread tiles of one image ("pixel block") and
//    `groups_per_cta` groups.  The input rows the block needs, for a chunk of
//    channels, are brought into shared memory by TMA (4-D tiled box, zero
//    fill outside the image = the padding) or, when the TMA stride rule
//    fails, by cp.async with zero fill; NSTAGE-deep ring.
//  * Accumulation (a5): per channel the thread loads its (T+2) x (S+2) input
//    window into registers once (128-bit LDS), then for every nonzero of its
//    group in that channel a warp-uniform switch on `id` issues T*S FFMAs
//    with static register indices.  Unstructured sparsity is not a dense
//    contraction, so this is CUDA-core FP32 (no tensor cores).
//  * Epilogue (a6): + bias, store; or ReLU + 2x2 max + first-max argmax
//    (the conv output is never written).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>

#include "spconv_internal.h"

namespace spconv {
namespace {

constexpr int TT = 2;     // output rows per thread tile
constexpr int TS = 4;     // output cols per thread tile
constexpr int NSTAGE = 3; // pipeline depth
constexpr int MAX_GPC = 8;

struct TiledArgs {
    const float *x;
    float *y;
    int32_t *argmax;
    const float *bias;
    const int32_t *group_rows;
    const int32_t *segoff;
    const TapEntry *stream;
    int N, C, H, W, F, Ho, Wo, Po, Qo;
    int tiles_x, tiles_per_img, blocks_per_img;
    int rows_staged, pitch, cc, stage_words;
    uint32_t box_bytes; // TMA transaction bytes per stage (cc * rows_staged * pitch * 4)
    int gpc, num_groups, num_gsets;
    int vec_store;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_u32(bar);
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void tma_load_4d(const CUtensorMap *map, uint64_t *bar, void *dst, int c0,
                                            int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void cp_async_4(void *dst, const void *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The warp-uniform tap dispatcher (inline-PTX threaded code, one brx.idx
// jump table; see gen_dispatch.py).  SPC_DISPATCH_R<R>(acc, xr, ptr) walks the
// stream at `ptr` until the sentinel id R*9 and leaves ptr past it.
#include "dispatch_gen.inc"

template <int R, bool FUSED, bool TMA>
__global__ void __launch_bounds__(32 * MAX_GPC, 2)
    tiled_kernel(const __grid_constant__ CUtensorMap tmap, const TiledArgs a) {
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t full_bar[NSTAGE];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int bid = blockIdx.x;
    const int gs = bid % a.num_gsets;
    bid /= a.num_gsets;
    const int pb = bid % a.blocks_per_img;
    const int n = bid / a.blocks_per_img;
    const int g = gs * a.gpc + warp;
    const bool group_ok = g < a.num_groups;

    const int q0 = pb * 32;
    const int ty0 = q0 / a.tiles_x;
    const int q = q0 + lane;
    const bool tile_ok = q < a.tiles_per_img;
    const int qq = tile_ok ? q : q0;
    const int ty = qq / a.tiles_x, tx = qq - (qq / a.tiles_x) * a.tiles_x;
    const int xoff = (ty - ty0) * TT * a.pitch + tx * TS;
    const int row0 = ty0 * TT - 1; // first staged input row (pad = 1)
    const int nchunks = (a.C + a.cc - 1) / a.cc;

    auto issue_chunk = [&](int k) {
        const int stage = k % NSTAGE;
        float *dst = smem + stage * a.stage_words;
        const int c0 = k * a.cc;
        if constexpr (TMA) {
            if (threadIdx.x == 0) {
                mbar_expect_tx(&full_bar[stage], a.box_bytes);
                tma_load_4d(&tmap, &full_bar[stage], dst, -1, row0, c0, n);
            }
        } else {
            const int per_c = a.rows_staged * a.pitch;
            const int cnt = min(a.cc, a.C - c0) * per_c;
            const float *xn = a.x + (size_t)n * a.C * a.H * a.W;
            for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
                const int cl = e / per_c;
                const int rem = e - cl * per_c;
                const int r = rem / a.pitch, col = rem - r * a.pitch;
                const int iy = row0 + r, ix = col - 1;
                const bool ok = iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
                const float *src = ok ? xn + ((size_t)(c0 + cl) * a.H + iy) * a.W + ix : a.x;
                cp_async_4(dst + e, src, ok);
            }
            cp_async_commit();
        }
    };

    if constexpr (TMA) {
        if (threadIdx.x == 0) {
            for (int s = 0; s < NSTAGE; ++s) mbar_init(&full_bar[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    for (int k = 0; k < NSTAGE - 1; ++k) {
        if (k < nchunks) issue_chunk(k);
        else if constexpr (!TMA) cp_async_commit();
    }

    float acc[R][TT][TS];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int t = 0; t < TT; ++t)
#pragma unroll
            for (int s = 0; s < TS; ++s) acc[r][t][s] = 0.0f;

    const int32_t *seg = a.segoff + (size_t)(group_ok ? g : 0) * (a.C + 1);

    for (int k = 0; k < nchunks; ++k) {
        const int stage = k % NSTAGE;
        // refill the stage consumed in iteration k-1 (all warps passed the barrier below)
        if (k + NSTAGE - 1 < nchunks) issue_chunk(k + NSTAGE - 1);
        else if constexpr (!TMA) cp_async_commit();
        if constexpr (TMA) {
            mbar_wait(&full_bar[stage], (k / NSTAGE) & 1);
        } else {
            cp_async_wait<NSTAGE - 1>();
            __syncthreads();
        }
        const int c0 = k * a.cc;
        const int cend = min(a.C, c0 + a.cc);
        const float *xs_stage = smem + stage * a.stage_words + xoff;
        if (group_ok) {
#pragma unroll 1
            for (int c = c0; c < cend; ++c) {
                const int e_beg = __ldg(seg + c), e_end = __ldg(seg + c + 1);
                if (e_end - e_beg <= 1) continue; // only the sentinel: no tap in this channel
                const float *xs = xs_stage + (c - c0) * a.rows_staged * a.pitch;
                float xr[TT + 2][TS + 2];
#pragma unroll
                for (int i = 0; i < TT + 2; ++i) {
                    const float4 p = *reinterpret_cast<const float4 *>(xs + i * a.pitch);
                    const float2 u = *reinterpret_cast<const float2 *>(xs + i * a.pitch + 4);
                    xr[i][0] = p.x; xr[i][1] = p.y; xr[i][2] = p.z; xr[i][3] = p.w;
                    xr[i][4] = u.x; xr[i][5] = u.y;
                }
                uint64_t sp = reinterpret_cast<uint64_t>(a.stream + e_beg);
                if constexpr (R == 8) {
                    SPC_DISPATCH_R8(acc, xr, sp);
                } else {
                    SPC_DISPATCH_R4(acc, xr, sp);
                }
            }
        }
        __syncthreads(); // stage may be overwritten by the next issue
    }

    if (!group_ok || !tile_ok) return;
    const int oy0 = ty * TT, ox0 = tx * TS;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int f = __ldg(a.group_rows + g * R + r);
        if (f < 0) continue;
        const float b = __ldg(a.bias + f);
        if constexpr (!FUSED) {
            float *yp = a.y + ((size_t)n * a.F + f) * a.Ho * a.Wo;
#pragma unroll
            for (int t = 0; t < TT; ++t) {
                const int oy = oy0 + t;
                if (oy >= a.Ho) continue;
                float o[TS];
#pragma unroll
                for (int s = 0; s < TS; ++s) o[s] = __fadd_rn(acc[r][t][s], b);
                float *row = yp + (size_t)oy * a.Wo + ox0;
                if (a.vec_store && ox0 + TS <= a.Wo) {
                    *reinterpret_cast<float4 *>(row) = make_float4(o[0], o[1], o[2], o[3]);
                } else {
#pragma unroll
                    for (int s = 0; s < TS; ++s)
                        if (ox0 + s < a.Wo) row[s] = o[s];
                }
            }
        } else {
            const int py = oy0 >> 1;
            if (py >= a.Po) continue;
            float *yp = a.y + ((size_t)n * a.F + f) * a.Po * a.Qo + (size_t)py * a.Qo;
            int32_t *ap = a.argmax ? a.argmax + ((size_t)n * a.F + f) * a.Po * a.Qo + (size_t)py * a.Qo
                                   : nullptr;
#pragma unroll
            for (int k2 = 0; k2 < TS / 2; ++k2) {
                const int px = (ox0 >> 1) + k2;
                if (px >= a.Qo) continue;
                float best = 0.0f;
                int bidx = 0;
#pragma unroll
                for (int w = 0; w < 4; ++w) { // row-major window order
                    const int dy = w >> 1, dx = w & 1;
                    const float v = __fadd_rn(acc[r][dy][2 * k2 + dx], b);
                    const float rv = v > 0.0f ? v : 0.0f;
                    if (w == 0 || rv > best) {
                        best = rv;
                        bidx = (oy0 + dy) * a.Wo + ox0 + 2 * k2 + dx;
                    }
                }
                yp[px] = best;
                if (ap) ap[px] = bidx;
            }
        }
    }
}

template <int R, bool FUSED, bool TMA>
cudaError_t launch_one(const CUtensorMap &map, const TiledArgs &a, int grid, size_t smem,
                       cudaStream_t s) {
    auto kern = tiled_kernel<R, FUSED, TMA>;
    // Opt in to the dynamic shared memory this launch needs (the attribute must not
    // exceed 227 KB minus the kernel's static shared memory); cached per device.
    static size_t attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    size_t &done = attr_done[dev & 63];
    if (smem > 48 * 1024 && __atomic_load_n(&done, __ATOMIC_ACQUIRE) < smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        __atomic_store_n(&done, smem, __ATOMIC_RELEASE);
    }
    kern<<<grid, 32 * a.gpc, smem, s>>>(map, a);
    return cudaGetLastError();
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

} // namespace

bool tiled_supported(int C, int H, int W, int F, int K, int stride, int pad) {
    (void)C; (void)F;
    return K == 3 && stride == 1 && pad == 1 && H >= 1 && W >= 1 && W + 8 <= 4096;
}

// The tiled kernel's staging ring must fit the device's opt-in shared memory (very wide
// rows do not: W = 3300 needs ~238 KB); checked at create so AUTO can fall back to the
// generic kernel instead of failing every forward.
bool tiled_fits(int C, int H, int W, int F, int K, int stride, int pad, int device) {
    if (!tiled_supported(C, H, W, F, K, stride, pad)) return false;
    Plan tmp;
    tmp.C = C; tmp.H = H; tmp.W = W; tmp.F = F; tmp.K = K; tmp.stride = stride; tmp.pad = pad;
    tmp.Ho = (H + 2 * pad - K) / stride + 1;
    tmp.Wo = (W + 2 * pad - K) / stride + 1;
    tmp.R = 4;
    tmp.num_groups = (F + 3) / 4;
    tiled_geometry(tmp);
    int optin = 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) {
        cudaGetLastError();
        optin = 227 * 1024;
    }
    return tmp.geo.smem_bytes + 1024 <= size_t(optin); // + the kernel's static barriers
}

int tiled_default_R(int C, int F, double density) {
    (void)C; (void)density;
    return F >= 8 ? 8 : 4;
}

void tiled_geometry(Plan &p) {
    TiledGeometry &g = p.geo;
    g.R = p.R;
    g.T = TT;
    g.S = TS;
    g.tiles_x = (p.Wo + TS - 1) / TS;
    g.tiles_y = (p.Ho + TT - 1) / TT;
    g.tiles_per_img = g.tiles_x * g.tiles_y;
    g.blocks_per_img = (g.tiles_per_img + 31) / 32;
    int span = 1;
    for (int pb = 0; pb < g.blocks_per_img; ++pb) {
        const int q0 = pb * 32, q1 = std::min(q0 + 31, g.tiles_per_img - 1);
        span = std::max(span, q1 / g.tiles_x - q0 / g.tiles_x + 1);
    }
    g.rows_staged = span * TT + 2;
    // pitch: >= W + 2 (one halo column each side), >= tiles_x*S + 4 (second 128-bit
    // load of the last tile), multiple of 4 (TMA box / 16-byte LDS), and
    // T*pitch/4 == tiles_x (mod 8) so the lanes of a quarter-warp that wrap to the
    // next tile row still hit distinct 16-byte bank groups.
    int base = std::max(p.W + 2, g.tiles_x * TS + 4);
    base = (base + 3) & ~3;
    g.pitch = base;
    for (int cand = base; cand < base + 64; cand += 4) {
        if (((TT * cand / 4 - g.tiles_x) % 8 + 8) % 8 == 0) {
            g.pitch = cand;
            break;
        }
    }
    const int per_c_bytes = g.rows_staged * g.pitch * 4;
    int cc = std::max(1, (24 * 1024) / per_c_bytes);
    cc = std::min(cc, p.C);
    // prefer a divisor of C close to cc (no ragged last chunk)
    for (int d = cc; d >= 1; --d)
        if (p.C % d == 0) {
            if (d * 2 >= cc) cc = d;
            break;
        }
    g.cc = cc;
    g.nstage = NSTAGE;
    int stage_words = cc * g.rows_staged * g.pitch;
    stage_words = (stage_words + 31) & ~31; // 128-byte aligned stages
    g.smem_bytes = size_t(NSTAGE) * stage_words * 4;
    g.groups_per_cta = std::min(p.num_groups, MAX_GPC);
    g.num_gsets = (p.num_groups + g.groups_per_cta - 1) / g.groups_per_cta;
    g.tma_ok = (p.W * 4) % 16 == 0 && g.pitch <= 256 && g.rows_staged <= 256 && cc <= 256;
}

cudaError_t launch_tiled(const Plan &p, int N, const float *x, float *y, int32_t *argmax,
                         bool fused, cudaStream_t s) {
    const TiledGeometry &g = p.geo;
    TiledArgs a;
    a.x = x; a.y = y; a.argmax = argmax;
    a.bias = p.d_bias; a.group_rows = p.d_group_rows; a.segoff = p.d_segoff; a.stream = p.d_stream;
    a.N = N; a.C = p.C; a.H = p.H; a.W = p.W; a.F = p.F; a.Ho = p.Ho; a.Wo = p.Wo;
    a.Po = p.Ho / 2; a.Qo = p.Wo / 2;
    a.tiles_x = g.tiles_x; a.tiles_per_img = g.tiles_per_img; a.blocks_per_img = g.blocks_per_img;
    a.rows_staged = g.rows_staged; a.pitch = g.pitch; a.cc = g.cc;
    a.stage_words = int(g.smem_bytes / 4 / NSTAGE);
    a.box_bytes = uint32_t(g.cc) * g.rows_staged * g.pitch * 4u;
    a.gpc = g.groups_per_cta; a.num_groups = p.num_groups; a.num_gsets = g.num_gsets;
    a.vec_store = (p.Wo % 4 == 0) && ((reinterpret_cast<uintptr_t>(y) & 15) == 0);
    const int64_t grid64 = (int64_t)N * g.blocks_per_img * g.num_gsets;
    if (grid64 > 0x7fffffff) return cudaErrorInvalidConfiguration;
    const int grid = int(grid64);

    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    // TMA tile loads need a 16-byte-aligned innermost start coordinate (probe:
    // scripts/probes/tma_probe.cu); this kernel stages from ix = -1, so it uses cp.async.
    bool use_tma = false && g.tma_ok && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    if (use_tma) {
        auto enc = get_encode();
        if (!enc) {
            use_tma = false;
        } else {
            cuuint64_t dims[4] = {(cuuint64_t)p.W, (cuuint64_t)p.H, (cuuint64_t)p.C, (cuuint64_t)N};
            cuuint64_t strides[3] = {(cuuint64_t)p.W * 4, (cuuint64_t)p.H * p.W * 4,
                                     (cuuint64_t)p.C * p.H * p.W * 4};
            cuuint32_t box[4] = {(cuuint32_t)g.pitch, (cuuint32_t)g.rows_staged, (cuuint32_t)g.cc, 1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(x), dims,
                             strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) use_tma = false;
        }
    }
    const size_t smem = g.smem_bytes;
#define SPC_LAUNCH(RR)                                                                          \
    if (p.R == RR) {                                                                            \
        if (fused) return use_tma ? launch_one<RR, true, true>(map, a, grid, smem, s)           \
                                  : launch_one<RR, true, false>(map, a, grid, smem, s);         \
        return use_tma ? launch_one<RR, false, true>(map, a, grid, smem, s)                     \
                       : launch_one<RR, false, false>(map, a, grid, smem, s);                   \
    }
    SPC_LAUNCH(8)
    SPC_LAUNCH(4)
#undef SPC_LAUNCH
    return cudaErrorInvalidValue;
}

} // namespace spconv
