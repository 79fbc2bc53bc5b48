// spconv_internal.h — plan layout shared by the C-ABI (spconv_api.cu) and the
// kernels (kernel_generic.cu, kernel_tiled.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "spconv.h"

namespace spconv {

// Packed decoded tap for the generic kernel:
// bits [31:6] = c, [5:3] = ky, [2:0] = kx  (K <= 8).
__host__ __device__ inline uint32_t pack_tap(int c, int ky, int kx) {
    return (uint32_t(c) << 6) | (uint32_t(ky) << 3) | uint32_t(kx);
}

// Tiled-kernel stream entry: one nonzero of a row group, in the order the
// kernel consumes it (channel-major, then case id ascending).
struct TapEntry {
    float v;    // filter value (bit-exact copy of values[j])
    int32_t id; // r * 9 + ky * 3 + kx  (r = slot of the output channel in its group); R*9 = end
};

struct TiledGeometry {
    int R, T, S;        // rows per group, output rows / cols per thread tile
    int tiles_x, tiles_y, tiles_per_img;
    int blocks_per_img; // ceil(tiles_per_img / 32)
    int rows_staged;    // RB: input rows staged per pixel block (max over blocks)
    int pitch;          // smem words per staged input row (>= W + 2, multiple of 4)
    int cc;             // channels per pipeline stage
    int nstage;         // pipeline depth
    int groups_per_cta; // GPC: one warp per group
    int num_gsets;      // ceil(num_groups / GPC)
    bool tma_ok;        // W * 4 % 16 == 0 (TMA global stride rule)
    size_t smem_bytes;
};

// Geometry of the warp-specialised pipeline kernel (kernel_pipe.cu) for one
// staging path: TMA (xs = 3: tile columns start at 4*tx - 3 so that the
// 16-byte-aligned TMA box start ix = -4 puts each window on a 16-byte smem
// boundary) or cp.async (xs = 0: the box starts at ix = -1).
struct PipeGeometry {
    bool ok = false;
    int xs;                  // column shift of the thread tiles (3: TMA, 0: cp.async)
    int T, S;                // thread tile: T output rows x S output columns
    int tiles_x, tiles_y;    // 4x4 thread tiles per image row / column
    int ipb, tr;             // images (band: tile-row bands) per block, tile rows per block (per image)
    int band;                // 1: blocks are ipb one-tile-row bands of the flattened (image, tile row) sequence
    int lanes;               // active lanes per consumer warp = ipb * tr * tiles_x
    int blocks_y;            // blocks per image (ipb == 1) along the tile rows
    int rs;                  // staged input rows per image = 4 * tr + 2
    int pitch;               // smem words per staged row (multiple of 4)
    int nstage;              // pipeline depth
    int cc, nchunks;         // input channels per stage, stages per pass
    int in_words;            // words of one stage's input box = ipb * rs * pitch
    int in_pad;              // bytes reserved for it (128-byte multiple)
    int st_bytes;            // bytes reserved per stage for the stream chunk
    size_t smem_bytes;       // dynamic shared memory per CTA
};

struct Plan {
    int C, H, W, F, K, stride, pad, Ho, Wo;
    int64_t nnz;
    int device;
    int kernel; // SPCONV_KERNEL_GENERIC or SPCONV_KERNEL_TILED
    // device copies (generic path)
    int32_t *d_rowptr = nullptr;
    uint32_t *d_taps = nullptr;
    float *d_values = nullptr;
    float *d_bias = nullptr; // always F floats (zeros when bias == NULL)
    // host copies for spconv_debug_decoded
    std::vector<int32_t> h_c, h_dy, h_dx;
    // tiled path
    int R = 0, num_groups = 0;
    int32_t *d_group_rows = nullptr; // [num_groups * R], -1 = empty slot
    int32_t *d_segoff = nullptr;     // [num_groups * (C + 1)] offsets into d_stream
    TapEntry *d_stream = nullptr;    // [nnz + num_groups*C]: per (group, channel) taps + sentinel
    TiledGeometry geo{};
    // pipeline (v2) path: GPC consumer warps per CTA, one row group each
    int gpc = 0, num_gsets = 0;
    int max_chunk_bytes = 0;       // largest (gset, stage) stream chunk incl. header
    int pipe_cc = 1;               // input channels per pipeline stage
    int pipe_dispatch = 0;         // 0: brx.idx threaded code (default), 1: tap-mask walk
    int32_t *d_chunk_start = nullptr; // [num_gsets * (nchunks + 1)] byte offsets into d_stream2
    uint4 *d_stream2 = nullptr;    // chunks: header (GPC u32 byte offsets) + 16-byte entries
    PipeGeometry pipe_tma{}, pipe_pad{}, pipe_cp{};
    int64_t device_bytes = 0;
    // spconv_forward_host staging
    std::mutex host_mu;
    float *d_xbuf = nullptr, *d_ybuf = nullptr;
    int32_t *d_abuf = nullptr;
    size_t xbuf_elems = 0, ybuf_elems = 0;
    // stream-K workspaces of the pipe kernel, one per stream (kept across calls so
    // consecutive launches are adjacent in the stream: programmatic dependent launch)
    std::mutex sk_mu;
    std::vector<std::pair<cudaStream_t, std::pair<void *, size_t>>> sk_ws;
    cudaStream_t host_stream = nullptr;    // host -> device copies
    static constexpr int HOST_KSTREAMS = 3;
    cudaStream_t host_kstream[HOST_KSTREAMS] = {}; // forwards of spconv_forward_host (chunks round-robin)
    cudaStream_t host_ostream = nullptr;   // device -> host copies
    static constexpr int MAX_HOST_CHUNKS = 16;
    cudaEvent_t host_ev_in[MAX_HOST_CHUNKS] = {}, host_ev_k[MAX_HOST_CHUNKS] = {};
};

// kernel_generic.cu
cudaError_t launch_generic_conv(const Plan &p, int N, const float *x, float *y, cudaStream_t s,
                                const float *res = nullptr, int epi = 0);
cudaError_t launch_generic_fused(const Plan &p, int N, const float *x, float *y, int32_t *argmax,
                                 cudaStream_t s);

// kernel_pipe.cu: keep the default stream-ordered pool's freed blocks cached
void keep_pool_cached();

// kernel_resize.cu
cudaError_t launch_resize(const float *x, float *y, int64_t planes, int Hin, int Win, int Hout, int Wout,
                          cudaStream_t s);

// kernel_pipe.cu
bool pipe_supported(int C, int H, int W, int F, int K, int stride, int pad);
void pipe_geometry(const Plan &p, int mode, PipeGeometry &g); // mode: 0 TMA, 1 TMA on padded copy, 2 cp.async
cudaError_t launch_pipe(const Plan &p, int N, const float *x, float *y, int32_t *argmax,
                        bool fused, cudaStream_t s, const float *res = nullptr, int epi = 0);

// kernel_tiled.cu
bool tiled_supported(int C, int H, int W, int F, int K, int stride, int pad);
int tiled_default_R(int C, int F, double density);
void tiled_geometry(Plan &p); // fills p.geo for p.R
cudaError_t launch_tiled(const Plan &p, int N, const float *x, float *y, int32_t *argmax,
                         bool fused, cudaStream_t s);

} // namespace spconv

// The opaque handle type of the public ABI is the plan itself.
struct spconv_plan_s : public spconv::Plan {};
