// spconv_internal.h — plan layout shared by the C-ABI (spconv_api.cu) and the
// kernels (kernel_generic.cu, kernel_tiled.cu).  Not part of the public ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstring>

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
    int lane_order = 0;      // lane -> tile: 0 slot-major, 1 tile-row-major (kernel_pipe.cu lane_tile)
    int colblocks = 1;       // wide rows: column blocks per tile row (units of their own)
    int cb_tiles = 0;        // tiles per column block (the block's lanes add one overlap tile)
    int tiles_total = 0;     // tiles per output row
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

// Debug / A/B knobs of the pipe kernel, read from the environment ONCE, when the
// plan is created (no getenv on the forward path).
struct PipeKnobs {
    int staging = -1;     // SPCONV_PIPE_STAGING: -1 auto, 1 padded copy, 2 cp.async
    int sk = -1;          // SPCONV_PIPE_SK: -1 auto, 0 off, 1 on (when there are more units than CTAs)
    int rev = 0;          // SPCONV_PIPE_REV=1: reversed work order (debug)
    int sk_split = 1;     // SPCONV_PIPE_SK_SPLIT: 1 per-warp cost-balanced split points (sk_split), 0 uniform
    int pdl = 1;          // SPCONV_PDL=0: launch without programmatic dependent launch
    char trace[256] = {}; // SPCONV_PIPE_TRACE=<file>: per-CTA timestamps (debug, synchronises)
    char prof[256] = {};  // SPCONV_PIPE_PROF=<file>: phase clock sums (-DSPC_PROF builds only)
    int debug = 0;        // SPCONV_DEBUG=1: plan self-check at create, synchronise + check every call
    int dense_stage = 0;  // SPCONV_DENSE_STAGE_BYTES: dense kernel input + weight bytes per stage (A/B)
};
void read_pipe_knobs(PipeKnobs &k);

// Geometry of the dense FP32 direct-conv kernel (kernel_dense.cu, NEXT-1).
struct DenseGeometry {
    bool ok = false;
    int S = 0;                // lane tile columns (7 or 8); rows are 2
    int LR = 0, LY = 0;       // lanes per staged row, lane rows per warp
    int RY = 0;               // lane rows per image = ceil(Ho / 2)
    int ipb = 0, bpi = 0;     // images per unit (small images) / units per image
    int rows = 0;             // staged rows per image slot (incl. the 2 halo rows)
    int pitch = 0;            // smem words per staged row (bank-conflict-free choice)
    int cc = 0, nchunks = 0, nstage = 0;
    int in_bytes = 0, w_bytes = 0, stage_bytes = 0;
    int fsets = 0;            // 64-output-channel sets
    int padded = 0, wq = 0;   // TMA on a right-padded copy (row stride not 16-byte aligned), its row length
    int xoff = 0;             // smem column of image column 0
    size_t smem_bytes = 0;
};

// Small per-plan caches of per-call host work (verdict r1 item 6): TMA descriptors keyed
// by (source pointer, N, geometry) and device-pointer validations keyed by pointer.
struct CallCache {
    std::mutex mu;
    struct Map {
        const void *src = nullptr;
        int N = 0;
        const void *geo = nullptr;
        CUtensorMap map;
    };
    Map maps[8];
    int next_map = 0;
    const void *valid[16] = {};
    int next_valid = 0;
    bool find_map(const void *src, int N, const void *geo, CUtensorMap &out) {
        std::lock_guard<std::mutex> lk(mu);
        for (auto &m : maps)
            if (m.src == src && m.N == N && m.geo == geo && src) {
                out = m.map;
                return true;
            }
        return false;
    }
    void put_map(const void *src, int N, const void *geo, const CUtensorMap &map) {
        std::lock_guard<std::mutex> lk(mu);
        maps[next_map] = Map{src, N, geo, map};
        next_map = (next_map + 1) % 8;
    }
    bool is_valid(const void *ptr) {
        std::lock_guard<std::mutex> lk(mu);
        for (const void *v : valid)
            if (v == ptr && ptr) return true;
        return false;
    }
    void put_valid(const void *ptr) {
        std::lock_guard<std::mutex> lk(mu);
        valid[next_valid] = ptr;
        next_valid = (next_valid + 1) % 16;
    }
};

struct Plan {
    int C, H, W, F, K, stride, pad, Ho, Wo;
    int64_t nnz;
    int device;
    int kernel; // SPCONV_KERNEL_GENERIC, _TILED or _PIPE (conv-only calls of a dense plan: see `dense`)
    bool auto_kernel = false; // created with SPCONV_KERNEL_AUTO (small calls may take the generic kernel)
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
    PipeGeometry pipe7_tma{}, pipe7_pad{}; // 7x4 tiles for non-fused calls (7-row tiles cover the height better)
    PipeKnobs knobs{};
    CallCache cache;
    // dense path (NEXT-1): conv-only calls of a plan whose kernel is SPCONV_KERNEL_DENSE
    // run the dense kernel on the densified filters; fused / epilogue calls use the pipe
    bool dense = false;
    float *d_wdense = nullptr;
    DenseGeometry dense_geo{};
    int64_t device_bytes = 0;
    // spconv_forward_host staging
    std::mutex host_mu;
    float *d_xbuf = nullptr, *d_ybuf = nullptr;
    int32_t *d_abuf = nullptr;
    size_t xbuf_elems = 0, ybuf_elems = 0;
    // stream-K workspaces of the pipe kernel, one per stream (kept across calls so
    // consecutive launches are adjacent in the stream: programmatic dependent launch)
    std::mutex sk_mu;
    struct SkSlot {
        cudaStream_t stream = nullptr;
        void *ptr = nullptr;
        size_t bytes = 0;
        unsigned seq = 0; // launches on this workspace: the counter slot of launch k is k % kSkSlots
    };
    std::vector<SkSlot> sk_ws;
    // AUTO plans of the pipe kernel at R = 4 and density >= kAltMinDensity also hold the
    // same layer at R = 2 (a complete plan of its own): per call, AUTO takes it when its
    // predicted time is lower -- 1.5x the warps per SM and shorter units, worth it when
    // the R = 4 units leave SMs idle (spconv_api.cu prefer_alt)
    Plan *alt = nullptr;
    double density = 0.0;
    // per-warp stream-K split tables (kernel_pipe.cu sk_split), cached per launch shape
    // (under sk_mu): a table depends on the units (N, geometry), the grid and the epilogue
    std::vector<float> sk_cost; // [gset][warp][C]: walk cost of the warp's group in channel c (tap units)
    struct SkTable {
        int N = -1, grid = 0, fused = 0;
        const void *geo = nullptr;
        std::vector<int32_t> unit;  // [grid + 1]: unit of boundary b
        std::vector<uint16_t> ch;   // [(grid + 1) * gpc]: per warp, the split channel in that unit
    };
    SkTable sk_tab[4];
    int sk_tab_next = 0;
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

// kernel_pipe.cu: the launch schedule of one forward (spconv_launch_info reports it)
struct PipeSchedule {
    int mode = 0;                       // 0 TMA on x, 1 TMA on a left-padded copy, 2 cp.async
    const PipeGeometry *g = nullptr;
    int64_t nunits = 0;                 // (pixel block, group set) work units
    int grid = 0;                       // persistent CTAs
    bool sk = false;                    // ordered stream-K split of the units over the CTAs
    int launches = 1;                   // kernel launches per call
};
bool pipe_schedule(const Plan &p, int N, uintptr_t x, PipeSchedule &q, bool conv_only, int epi = 0);
// per-warp stream-K split table of that schedule (kernel_pipe.cu); unit / ch may be null
bool sk_table(const Plan &p, const PipeSchedule &q, int N, bool fused, int32_t *unit, uint16_t *ch);
// the split itself, from per-(gset, warp, channel) costs (plan-free: spconv_debug_sk_split)
void sk_split_core(const float *lane_cost, int C, int gpc, int ngs, int num_groups, int cc, int64_t U, int G, bool fused,
                   std::vector<int32_t> &unit_out, std::vector<uint16_t> &ch_out);
// Stream-K workspace of one launch (kernel_pipe.cu, shared by the dense kernel).
constexpr size_t kSkHeader = 32768; // counter slots, then u64 flags; partial sums after
constexpr int kSkSlots = 64;         // [ticket, finished] pairs, one per launch modulo 64
constexpr size_t kSkFlags = kSkSlots * 8; // byte offset of the flags
// per-warp split tables travel in the kernel parameters: up to kSkTabCta CTAs and
// kSkTabGpc warps per CTA (4.5 KB); larger grids use the uniform channel split
constexpr double kAltMinDensity = 0.08;
constexpr int kSkTabCta = 160;
constexpr int kSkTabGpc = 12;
// walk cost model of the split (units of one tap case, ~125 SM cycles on B200), from
// per-CTA trace fits (profiles/r02/sk_split_*.txt; c2: a tap case 66 ns, a reload
// ~4.5 taps, a unit epilogue ~3.0 us conv / ~4.4 us fused): a window reload costs
// kSkReload taps, a channel of the stage loop kSkChan, and per CTA item a resume,
// a unit epilogue (conv / fused) or a park
constexpr double kSkReload = 4.5, kSkChan = 0.6, kSkResume = 20.0, kSkEpiConv = 45.0, kSkEpiFused = 50.0,
                 kSkPark = 25.0;
struct SkWorkspace {
    void *base = nullptr;
    bool async = false;                 // a per-call stream-ordered allocation (freed by release)
    std::unique_lock<std::mutex> lock;  // the plan's workspace lock, held until release
    unsigned *ticket = nullptr;
    unsigned long long *flag = nullptr;
    void *part = nullptr;
    cudaError_t release(cudaStream_t s);
};
cudaError_t stream_k_workspace(const Plan &p, cudaStream_t s, size_t part_bytes, int nflags, SkWorkspace &w);
unsigned long long next_sk_epoch();
int sm_count_of_current_device();

// kernel_pipe.cu
bool pipe_supported(int C, int H, int W, int F, int K, int stride, int pad);
// mode: 0 TMA, 1 TMA on padded copy, 2 cp.async; T: output rows per thread tile (8, or 7)
void pipe_geometry(const Plan &p, int mode, PipeGeometry &g, int T = 8);
cudaError_t launch_pipe(const Plan &p, int N, const float *x, float *y, int32_t *argmax,
                        bool fused, cudaStream_t s, const float *res = nullptr, int epi = 0);

// kernel_dense.cu.  AUTO routes every call on a layer at or above the break-even density
// to the dense kernel.  Measured B200 break-even of the sparse pipe kernel against it:
// 0.45 (c2 shape), 0.46 (c5), 0.77 (c4, where the dense geometry leaves lanes and SMs
// idle) -- profiles/r02/breakeven_*.jsonl; the paper's own CPU figure is
// 0.435.  So: 0.5 when the dense geometry's expected efficiency is high
// (>= 0.8: full lane tiles, every SM busy), else 0.75.
constexpr double kDenseBreakEven = 0.50, kDenseBreakEvenWeak = 0.75, kDenseGoodGeometry = 0.80;
bool dense_supported(int C, int H, int W, int F, int K, int stride, int pad);
void dense_geometry(const Plan &p, DenseGeometry &g);
std::vector<float> dense_weights(const Plan &p, const DenseGeometry &g, const std::vector<int32_t> &rowptr,
                                 const std::vector<int32_t> &colidx, const std::vector<float> &values);
cudaError_t launch_dense(const Plan &p, int N, const float *x, float *y, int32_t *argmax, bool fused,
                         cudaStream_t s, const float *res = nullptr, int epi = 0);
bool dense_stream_k(const Plan &p, int64_t nunits, int grid);
double dense_expected_efficiency(const Plan &p, int N);

// kernel_tiled.cu
bool tiled_supported(int C, int H, int W, int F, int K, int stride, int pad);
int tiled_default_R(int C, int F, double density);
bool tiled_fits(int C, int H, int W, int F, int K, int stride, int pad, int device);
void tiled_geometry(Plan &p); // fills p.geo for p.R
cudaError_t launch_tiled(const Plan &p, int N, const float *x, float *y, int32_t *argmax,
                         bool fused, cudaStream_t s);

} // namespace spconv

// The opaque handle type of the public ABI is the plan itself.
struct spconv_plan_s : public spconv::Plan {};
