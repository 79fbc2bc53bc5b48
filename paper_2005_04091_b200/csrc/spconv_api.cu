// spconv_api.cu — the C-ABI of include/spconv.h: plan creation (validate,
// decode, group, upload), argument checking and the
// kernel launches (a4-a6).  No CPU compute path exists: every output value is
// produced by a CUDA kernel (kernel_generic.cu / kernel_tiled.cu).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <numeric>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "spconv_internal.h"

using spconv::Plan;

namespace {

// Last CUDA error seen by an entry point on this thread (spconv_last_cuda_error).
thread_local cudaError_t g_last_cuda = cudaSuccess;

int cuda_fail(cudaError_t e) {
    g_last_cuda = e;
    return SPCONV_ERR_CUDA;
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Host copy of an array that may live in host or device memory.
template <typename T>
int fetch(const T *src, int64_t n, std::vector<T> &dst) {
    dst.resize(size_t(n));
    if (n == 0) return SPCONV_OK;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, src);
    if (e != cudaSuccess) {
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

template <typename T>
int upload(T **dptr, const T *src, size_t n, int64_t &bytes) {
    const size_t sz = sizeof(T) * std::max<size_t>(n, 1);
    if (cudaMalloc(reinterpret_cast<void **>(dptr), sz) != cudaSuccess) {
        cudaGetLastError();
        return SPCONV_ERR_OOM;
    }
    bytes += int64_t(sz);
    if (n && cudaMemcpy(*dptr, src, sizeof(T) * n, cudaMemcpyHostToDevice) != cudaSuccess)
        return SPCONV_ERR_CUDA;
    return SPCONV_OK;
}

void free_plan(Plan *p) {
    if (!p) return;
    free_plan(p->alt);
    DeviceGuard g(p->device);
    cudaFree(p->d_rowptr);
    cudaFree(p->d_taps);
    cudaFree(p->d_values);
    cudaFree(p->d_bias);
    cudaFree(p->d_group_rows);
    cudaFree(p->d_segoff);
    cudaFree(p->d_stream);
    cudaFree(p->d_chunk_start);
    cudaFree(p->d_stream2);
    cudaFree(p->d_wdense);
    for (auto &w : p->sk_ws) cudaFree(w.ptr);
    cudaFree(p->d_xbuf);
    cudaFree(p->d_ybuf);
    cudaFree(p->d_abuf);
    if (p->host_stream) cudaStreamDestroy(p->host_stream);
    for (cudaStream_t ks : p->host_kstream)
        if (ks) cudaStreamDestroy(ks);
    if (p->host_ostream) cudaStreamDestroy(p->host_ostream);
    for (int i = 0; i < Plan::MAX_HOST_CHUNKS; ++i) {
        if (p->host_ev_in[i]) cudaEventDestroy(p->host_ev_in[i]);
        if (p->host_ev_k[i]) cudaEventDestroy(p->host_ev_k[i]);
    }
    delete static_cast<spconv_plan_s *>(p);
}

// x/y/argmax must be device memory of the plan's device (no CPU fallback).
int check_device_ptr(const void *ptr, int device) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return SPCONV_ERR_DEVICE;
    }
    if (at.type == cudaMemoryTypeManaged) return SPCONV_OK;
    if (at.type != cudaMemoryTypeDevice || at.device != device) return SPCONV_ERR_DEVICE;
    return SPCONV_OK;
}

bool overlap(const void *a, size_t abytes, const void *b, size_t bbytes) {
    const char *a0 = static_cast<const char *>(a), *b0 = static_cast<const char *>(b);
    return a0 < b0 + bbytes && b0 < a0 + abytes;
}

// Row groups with balanced nnz: longest-processing-time-first into
// ceil(F/R) groups of at most R rows.
std::vector<int32_t> balance_groups(const std::vector<int32_t> &rowptr, int F, int R, int &ngroups) {
    ngroups = (F + R - 1) / R;
    std::vector<int> order(F);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return rowptr[a + 1] - rowptr[a] > rowptr[b + 1] - rowptr[b];
    });
    std::vector<int64_t> load(ngroups, 0);
    std::vector<int> fill(ngroups, 0);
    std::vector<int32_t> rows(size_t(ngroups) * R, -1);
    for (int f : order) {
        int best = -1;
        for (int g = 0; g < ngroups; ++g)
            if (fill[g] < R && (best < 0 || load[g] < load[best])) best = g;
        rows[size_t(best) * R + fill[best]++] = f;
        load[best] += rowptr[f + 1] - rowptr[f];
    }
    return rows;
}

// NVTX range over an entry point (SURVEY.md §5 tracing): visible in nsys / ncu
// timelines, a no-op without an attached tool.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// SPCONV_DEBUG=1 self-check of a built pipe plan (SURVEY.md §5 "extra validation"):
// walk every (group set, stage, warp) tap stream exactly as the kernel's dispatcher
// does and rebuild each output channel's (colidx, value) sequence from it; it must be
// the CSR row, in ascending colidx order (the FP32 contract), entry for entry.
bool pipe_stream_self_check(const Plan *p, const std::vector<uint4> &out, const std::vector<int32_t> &cstart,
                            const std::vector<int32_t> &grows, const std::vector<int32_t> &rowptr,
                            const std::vector<int32_t> &colidx, const std::vector<float> &values) {
    const int R = p->R, C = p->C, cc = p->pipe_cc, nch = (C + cc - 1) / cc;
    const uint32_t NEXT = uint32_t(R * 9), END = uint32_t(R * 9 + 1);
    std::vector<std::vector<std::pair<int, uint32_t>>> got(size_t(p->F));
    const char *base = reinterpret_cast<const char *>(out.data());
    for (int gs = 0; gs < p->num_gsets; ++gs)
        for (int j = 0; j < nch; ++j) {
            const int32_t c0b = cstart[size_t(gs) * (nch + 1) + j];
            const uint32_t *hdr = reinterpret_cast<const uint32_t *>(base + c0b);
            for (int w = 0; w < p->gpc; ++w) {
                const int g = gs * p->gpc + w;
                const uint2 *e = reinterpret_cast<const uint2 *>(base + c0b + hdr[w]);
                uint32_t cs = e[0].y; // lead entry: the case of entry 1
                int ch = j * cc;
                for (size_t k = 1;; ++k) {
                    if (cs == END) break;
                    if (cs == NEXT) {
                        if (e[k].x < 1) return false;
                        ch += int(e[k].x);
                    } else {
                        if (cs > NEXT || g >= p->num_groups || ch >= std::min(C, (j + 1) * cc)) return false;
                        const int r = int(cs) % R, tap = int(cs) / R;
                        const int f = grows[size_t(g) * R + r];
                        if (f < 0) return false;
                        got[size_t(f)].push_back({ch * 9 + tap, e[k].x});
                    }
                    cs = e[k].y;
                    if (k > size_t(4) * (size_t(R) * 9 + 2) * size_t(cc) + 8) return false; // runaway
                }
            }
        }
    for (int f = 0; f < p->F; ++f) {
        const auto &v = got[size_t(f)];
        if (int64_t(v.size()) != int64_t(rowptr[size_t(f) + 1]) - rowptr[size_t(f)]) return false;
        for (size_t i = 0; i < v.size(); ++i) {
            const int32_t j = rowptr[size_t(f)] + int32_t(i);
            uint32_t bits;
            std::memcpy(&bits, &values[size_t(j)], 4);
            if (v[i].first != colidx[size_t(j)] || v[i].second != bits) return false;
        }
    }
    return true;
}

int build_plan(Plan *p, const std::vector<int32_t> &rowptr, const std::vector<int32_t> &colidx,
               const std::vector<float> &values, const std::vector<float> &bias, int rows_per_group) {
    const int K = p->K;
    // a2: decode colidx -> (c, ky, kx)
    std::vector<uint32_t> taps(size_t(p->nnz));
    p->h_c.resize(size_t(p->nnz));
    p->h_dy.resize(size_t(p->nnz));
    p->h_dx.resize(size_t(p->nnz));
    for (int64_t j = 0; j < p->nnz; ++j) {
        const int col = colidx[size_t(j)];
        const int c = col / (K * K), ky = (col / K) % K, kx = col % K;
        taps[size_t(j)] = spconv::pack_tap(c, ky, kx);
        p->h_c[size_t(j)] = c;
        p->h_dy[size_t(j)] = ky - p->pad;
        p->h_dx[size_t(j)] = kx - p->pad;
    }
    int st;
    if ((st = upload(&p->d_rowptr, rowptr.data(), rowptr.size(), p->device_bytes))) return st;
    if ((st = upload(&p->d_taps, taps.data(), taps.size(), p->device_bytes))) return st;
    if ((st = upload(&p->d_values, values.data(), values.size(), p->device_bytes))) return st;
    if ((st = upload(&p->d_bias, bias.data(), bias.size(), p->device_bytes))) return st;

    if (p->kernel == SPCONV_KERNEL_GENERIC) return SPCONV_OK;
    // a3: balanced row groups
    const int R = rows_per_group;
    p->R = R;
    std::vector<int32_t> grows = balance_groups(rowptr, p->F, R, p->num_groups);
    const int C = p->C;
    if (p->kernel == SPCONV_KERNEL_PIPE) {
        // Per (group set, pipeline stage of cc channels) chunk: a header of GPC u32
        // byte offsets (one per warp, 16-byte padded) then, per warp, for each channel
        // of the stage its group's nonzeros with case = (ky*3 + kx)*R + r, ascending
        // by case, followed by a "next channel" marker (case R*9) or, after the
        // stage's last channel, an "end" marker (R*9+1).  Stored as 8-byte entries
        // {v, case of the following entry} behind a lead entry {0, first case}
        // (gen_dispatch2.py), two per 16-byte stream word.
        // Ascending case within a channel, channels in order: every output row's
        // taps are consumed in ascending colidx order (the FP32 contract).
        // warps (= groups) per CTA: 8 at R = 4; at R = 2 up to 12, spread evenly over
        // the group sets (32 groups -> 3 sets of 11 warps, not 12 + 12 + 8)
        if (R == 2) {
            const int sets = (p->num_groups + 11) / 12;
            p->gpc = (p->num_groups + sets - 1) / sets;
        } else {
            p->gpc = std::min(p->num_groups, 8);
        }
        // brx.idx threaded code (default; measured faster on B200) or the tap-mask walk
        p->pipe_dispatch = 0;
        if (const char *e = std::getenv("SPCONV_PIPE_DISPATCH"))
            if (std::strcmp(e, "mask") == 0 && R == 4) p->pipe_dispatch = 1;
        p->num_gsets = (p->num_groups + p->gpc - 1) / p->gpc;
        const int hdr = ((p->gpc * 4 + 15) / 16) * 16;
        std::vector<uint4> out;
        // per group: per channel list of (case, value)
        std::vector<std::vector<std::vector<std::pair<int, float>>>> byc(size_t(p->num_groups));
        for (int g = 0; g < p->num_groups; ++g) {
            byc[size_t(g)].resize(size_t(C));
            for (int r = 0; r < R; ++r) {
                const int f = grows[size_t(g) * R + r];
                if (f < 0) continue;
                for (int32_t j = rowptr[f]; j < rowptr[f + 1]; ++j) {
                    const int col = colidx[size_t(j)];
                    const int c = col / 9, ky = (col / 3) % 3, kx = col % 3;
                    byc[size_t(g)][size_t(c)].push_back({(ky * 3 + kx) * R + r, values[size_t(j)]});
                }
            }
        }
        // walk cost of each (group set, warp, channel) for the stream-K split (sk_split)
        p->sk_cost.assign(size_t(p->num_gsets) * p->gpc * C, 0.0f);
        for (int g = 0; g < p->num_groups; ++g)
            for (int c = 0; c < C; ++c) {
                const size_t k = byc[size_t(g)][size_t(c)].size();
                p->sk_cost[size_t(g) * C + c] = float(double(k) + (k ? spconv::kSkReload : 0.0) + spconv::kSkChan);
            }
        // channels per stage: about 88 KB of staged input per stage (fewer stage
        // boundaries: each costs a barrier wait, a header load and a refill)
        p->pipe_cc = 1;
        p->max_chunk_bytes = 0;
        spconv::pipe_geometry(*p, 2, p->pipe_cp);
        spconv::pipe_geometry(*p, 1, p->pipe_pad);
        spconv::pipe_geometry(*p, 0, p->pipe_tma);
        const int per_ch = std::max({p->pipe_tma.in_words, p->pipe_pad.in_words, p->pipe_cp.in_words}) * 4;
        int stage_target = 90112; // measured on B200: c4 -1.5% vs 80 KB, c2/c3/c5 equal
        if (const char *e = std::getenv("SPCONV_PIPE_STAGE_BYTES")) stage_target = std::max(4096, std::atoi(e));
        const bool tma_feasible = p->pipe_tma.ok, pad_feasible = p->pipe_pad.ok;
        std::vector<int32_t> cstart;
        // the stream layout depends on cc; shrink cc until the ring fits shared memory
        for (int cc_try = std::max(1, std::min({32, C, stage_target / std::max(per_ch, 1)}));; cc_try /= 2) {
            // balanced chunks for the same chunk count (stage boundaries cost ~0.5 us
            // each on c2): a divisor of C when one gives that count
            const int nch_try = (C + cc_try - 1) / cc_try;
            int cc_eq = (C + nch_try - 1) / nch_try; // same chunk count, sizes within one channel
            for (int d = cc_eq; d <= cc_try; ++d)
                if (C % d == 0 && C / d == nch_try) { cc_eq = d; break; }
            if (const char *e = std::getenv("SPCONV_PIPE_CC")) // experiments: force the stage size
                cc_eq = std::max(1, std::min(cc_try, std::atoi(e)));
            p->pipe_cc = cc_eq;
            const int cc = p->pipe_cc, nchunks = (C + cc - 1) / cc;
            out.clear();
            const uint32_t NEXT = uint32_t(R * 9), END = uint32_t(R * 9 + 1);
            cstart.assign(size_t(p->num_gsets) * (nchunks + 1), 0);
            int maxb = 0;
            for (int gs = 0; gs < p->num_gsets; ++gs) {
                for (int j = 0; j < nchunks; ++j) {
                    const size_t base = out.size();
                    cstart[size_t(gs) * (nchunks + 1) + j] = int32_t(base * 16);
                    out.resize(base + size_t(hdr / 16));
                    std::vector<uint32_t> offs(size_t(p->gpc), 0);
                    const int c0 = j * cc, c1 = std::min(C, c0 + cc);
                    for (int w = 0; w < p->gpc; ++w) {
                        const int g = gs * p->gpc + w;
                        offs[size_t(w)] = uint32_t((out.size() - base) * 16);
                        if (p->pipe_dispatch == 1) {
                            // mask walk: per channel a 9R-bit mask (bit tap*R + r) then the
                            // values as (v, v) pairs in tap-major, row-minor order; 8-byte
                            // items packed into the 16-byte stream words
                            std::vector<uint64_t> items, dense;
                            for (int c = c0; c < c1; ++c) {
                                uint64_t m = 0;
                                std::vector<uint64_t> blk(size_t(9 * R), 0);
                                if (g < p->num_groups)
                                    for (auto &e : byc[size_t(g)][size_t(c)]) {
                                        const int r = e.first % R, tap = e.first / R;
                                        m |= uint64_t(1) << (tap * R + r);
                                        uint32_t bits;
                                        std::memcpy(&bits, &e.second, 4);
                                        blk[size_t(tap * R + r)] = (uint64_t(bits) << 32) | bits;
                                    }
                                items.push_back(m);
                                dense.insert(dense.end(), blk.begin(), blk.end());
                            }
                            if (items.size() & 1) items.push_back(0); // dense blocks start 16-byte aligned
                            items.insert(items.end(), dense.begin(), dense.end());
                            if (items.size() & 1) items.push_back(0);
                            for (size_t i = 0; i < items.size(); i += 2)
                                out.push_back(make_uint4(uint32_t(items[i]), uint32_t(items[i] >> 32),
                                                         uint32_t(items[i + 1]), uint32_t(items[i + 1] >> 32)));
                            continue;
                        }
                        // the walk order (case, value) of this warp's stage, then stored with
                        // each entry carrying the NEXT entry's case behind a lead entry, so the
                        // case id of k+2 is loaded while case k+1 is dispatched
                        // A "next channel" marker carries k (>= 1) in its value field: the walk
                        // skips channels without nonzeros for this group instead of reloading
                        // the window for each (the window starts at channel c0).
                        std::vector<std::pair<uint32_t, uint32_t>> walk;
                        int at = c0;
                        for (int c = c0; c < c1; ++c) {
                            if (g < p->num_groups && !byc[size_t(g)][size_t(c)].empty()) {
                                if (c > at) walk.push_back({NEXT, uint32_t(c - at)});
                                at = c;
                                auto v = byc[size_t(g)][size_t(c)];
                                std::stable_sort(v.begin(), v.end(),
                                                 [](const std::pair<int, float> &a, const std::pair<int, float> &b) {
                                                     return a.first < b.first;
                                                 });
                                for (auto &e : v) {
                                    uint32_t bits;
                                    std::memcpy(&bits, &e.second, 4);
                                    walk.push_back({uint32_t(e.first), bits});
                                }
                            }
                        }
                        walk.push_back({END, 0u});
                        // 8-byte entries {value, case of the next entry} behind a lead entry
                        // {0, first case}, two per 16-byte stream word (a segment is padded
                        // to a whole word)
                        std::vector<uint2> ent;
                        ent.push_back(make_uint2(0u, walk[0].first));
                        for (size_t k = 0; k < walk.size(); ++k)
                            ent.push_back(make_uint2(walk[k].second, k + 1 < walk.size() ? walk[k + 1].first : END));
                        if (ent.size() & 1) ent.push_back(make_uint2(0u, END));
                        for (size_t k = 0; k < ent.size(); k += 2)
                            out.push_back(make_uint4(ent[k].x, ent[k].y, ent[k + 1].x, ent[k + 1].y));
                    }
                    std::memcpy(reinterpret_cast<char *>(out.data() + base), offs.data(), offs.size() * 4);
                    maxb = std::max(maxb, int((out.size() - base) * 16));
                }
                cstart[size_t(gs) * (nchunks + 1) + nchunks] = int32_t(out.size() * 16);
            }
            if (out.size() * 16 > size_t(INT32_MAX)) return SPCONV_ERR_UNSUPPORTED;
            p->max_chunk_bytes = maxb;
            spconv::pipe_geometry(*p, 0, p->pipe_tma);
            spconv::pipe_geometry(*p, 1, p->pipe_pad);
            spconv::pipe_geometry(*p, 2, p->pipe_cp);
            if ((p->pipe_cp.ok && (p->pipe_tma.ok || !tma_feasible) && (p->pipe_pad.ok || !pad_feasible)) ||
                cc_try == 1)
                break;
        }
        // 7-row tiles for conv-only calls when they cover the image height better than
        // 8-row ones (c4 14x14, VGG 28x28: 100% vs 87.5% of the rows; the tap streams do
        // not depend on the tile shape, only the staging geometry does)
        const int t8 = (p->Ho + 7) / 8 * 8, t7 = (p->Ho + 6) / 7 * 7;
        if (p->pipe_dispatch == 0 && t7 < t8) {
            spconv::pipe_geometry(*p, 0, p->pipe7_tma, 7);
            spconv::pipe_geometry(*p, 1, p->pipe7_pad, 7);
        }
        if ((st = upload(&p->d_group_rows, grows.data(), grows.size(), p->device_bytes))) return st;
        if ((st = upload(&p->d_chunk_start, cstart.data(), cstart.size(), p->device_bytes))) return st;
        if (p->knobs.debug && p->pipe_dispatch == 0 &&
            !pipe_stream_self_check(p, out, cstart, grows, rowptr, colidx, values))
            return SPCONV_ERR_INTERNAL;
        if ((st = upload(&p->d_stream2, out.data(), out.size(), p->device_bytes))) return st;
        if (!p->pipe_cp.ok) return SPCONV_ERR_UNSUPPORTED;
        return SPCONV_OK;
    }
    // tiled (v1): per (group, channel) tap streams
    std::vector<int32_t> segoff(size_t(p->num_groups) * (C + 1));
    std::vector<spconv::TapEntry> stream;
    stream.reserve(size_t(p->nnz) + size_t(p->num_groups) * C);
    std::vector<std::vector<spconv::TapEntry>> bucket(C);
    for (int g = 0; g < p->num_groups; ++g) {
        for (auto &b : bucket) b.clear();
        for (int r = 0; r < R; ++r) {
            const int f = grows[size_t(g) * R + r];
            if (f < 0) continue;
            for (int32_t j = rowptr[f]; j < rowptr[f + 1]; ++j) {
                const int col = colidx[size_t(j)];
                const int c = col / 9, ky = (col / 3) % 3, kx = col % 3;
                bucket[c].push_back({values[size_t(j)], r * 9 + ky * 3 + kx});
            }
        }
        for (int c = 0; c < C; ++c) {
            segoff[size_t(g) * (C + 1) + c] = int32_t(stream.size());
            auto &b = bucket[c];
            std::stable_sort(b.begin(), b.end(),
                             [](const spconv::TapEntry &a, const spconv::TapEntry &b) { return a.id < b.id; });
            stream.insert(stream.end(), b.begin(), b.end());
            stream.push_back({0.0f, R * 9}); // sentinel: ends the channel's dispatch
        }
        segoff[size_t(g) * (C + 1) + C] = int32_t(stream.size());
    }
    if ((st = upload(&p->d_group_rows, grows.data(), grows.size(), p->device_bytes))) return st;
    if ((st = upload(&p->d_segoff, segoff.data(), segoff.size(), p->device_bytes))) return st;
    if ((st = upload(&p->d_stream, stream.data(), stream.size(), p->device_bytes))) return st;
    spconv::tiled_geometry(*p);
    return SPCONV_OK;
}

} // namespace

extern "C" {

const char *spconv_status_string(int status) {
    switch (status) {
        case SPCONV_OK: return "ok";
        case SPCONV_ERR_NULLPTR: return "required pointer is NULL";
        case SPCONV_ERR_SHAPE: return "invalid shape";
        case SPCONV_ERR_CSR: return "malformed CSR (rowptr/colidx/values)";
        case SPCONV_ERR_UNSUPPORTED: return "unsupported shape or option";
        case SPCONV_ERR_ALIGN: return "pointer not 4-byte aligned";
        case SPCONV_ERR_DEVICE: return "pointer is not device memory of the plan's device";
        case SPCONV_ERR_CUDA: return "CUDA error";
        case SPCONV_ERR_OOM: return "out of memory";
        case SPCONV_ERR_ALIAS: return "output overlaps input";
        case SPCONV_ERR_INTERNAL: return "plan self-check failed (SPCONV_DEBUG)";
        default: return "unknown status";
    }
}

int spconv_abi_version(void) { return SPCONV_ABI_VERSION; }

const char *spconv_last_cuda_error(void) {
    return g_last_cuda == cudaSuccess ? "no CUDA error" : cudaGetErrorString(g_last_cuda);
}

int spconv_create_ex(spconv_plan_t *plan, int C, int H, int W, int F, int K, int stride, int pad,
                     const int32_t *rowptr, const int32_t *colidx, const float *values, int64_t nnz,
                     const float *bias, int device, const spconv_options_t *opts) {
    NvtxRange nvtx("spconv_create");
    if (!plan) return SPCONV_ERR_NULLPTR;
    *plan = nullptr;
    if (!rowptr || (nnz > 0 && (!colidx || !values))) return SPCONV_ERR_NULLPTR;
    if (C < 1 || H < 1 || W < 1 || F < 1 || K < 1 || stride < 1 || pad < 0 || nnz < 0)
        return SPCONV_ERR_SHAPE;
    if (K > 8 || stride > 8 || pad > 16 || nnz > INT32_MAX || int64_t(C) * K * K > INT32_MAX / 2)
        return SPCONV_ERR_UNSUPPORTED;
    const int Hp = H + 2 * pad, Wp = W + 2 * pad;
    if (Hp < K || Wp < K) return SPCONV_ERR_SHAPE;
    spconv_options_t o{};
    if (opts) o = *opts;
    if (o.kernel < SPCONV_KERNEL_AUTO || o.kernel > SPCONV_KERNEL_DENSE) return SPCONV_ERR_UNSUPPORTED;
    for (int r : o.reserved)
        if (r != 0) return SPCONV_ERR_UNSUPPORTED;

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
        cudaGetLastError();
        return SPCONV_ERR_CUDA;
    }
    if (device < 0 || device >= ndev) return SPCONV_ERR_DEVICE;
    DeviceGuard guard(device);
    if (!guard.ok) return SPCONV_ERR_CUDA;

    // a1: validate (host copies; inputs may be host or device pointers)
    std::vector<int32_t> h_rowptr, h_colidx;
    std::vector<float> h_values, h_bias;
    int st;
    if ((st = fetch(rowptr, F + 1, h_rowptr))) return st;
    if ((st = fetch(colidx, nnz, h_colidx))) return st;
    if ((st = fetch(values, nnz, h_values))) return st;
    if (bias) {
        if ((st = fetch(bias, F, h_bias))) return st;
    } else {
        h_bias.assign(size_t(F), 0.0f);
    }
    if (h_rowptr[0] != 0 || int64_t(h_rowptr[size_t(F)]) != nnz) return SPCONV_ERR_CSR;
    const int32_t ncol = C * K * K;
    for (int f = 0; f < F; ++f) {
        const int32_t b = h_rowptr[size_t(f)], e = h_rowptr[size_t(f) + 1];
        if (e < b) return SPCONV_ERR_CSR;
        for (int32_t j = b; j < e; ++j) {
            const int32_t col = h_colidx[size_t(j)];
            if (col < 0 || col >= ncol) return SPCONV_ERR_CSR;
            if (j > b && col <= h_colidx[size_t(j) - 1]) return SPCONV_ERR_CSR; // sorted, unique
            if (!std::isfinite(h_values[size_t(j)])) return SPCONV_ERR_CSR;
        }
    }
    for (float b : h_bias)
        if (!std::isfinite(b)) return SPCONV_ERR_CSR;

    spconv_plan_s *p = new (std::nothrow) spconv_plan_s;
    if (!p) return SPCONV_ERR_OOM;
    p->C = C; p->H = H; p->W = W; p->F = F; p->K = K; p->stride = stride; p->pad = pad;
    p->Ho = (Hp - K) / stride + 1;
    p->Wo = (Wp - K) / stride + 1;
    p->nnz = nnz;
    p->device = device;
    spconv::read_pipe_knobs(p->knobs); // debug / A/B knobs: read once, here
    const bool tiled_ok = spconv::tiled_fits(C, H, W, F, K, stride, pad, device);
    const bool pipe_ok = spconv::pipe_supported(C, H, W, F, K, stride, pad);
    const bool dense_ok = spconv::dense_supported(C, H, W, F, K, stride, pad);
    if ((o.kernel == SPCONV_KERNEL_TILED && !tiled_ok) || (o.kernel == SPCONV_KERNEL_PIPE && !pipe_ok) ||
        (o.kernel == SPCONV_KERNEL_DENSE && !dense_ok)) {
        delete p;
        return SPCONV_ERR_UNSUPPORTED;
    }
    const double density = double(nnz) / (double(F) * ncol);
    p->density = density;
    p->auto_kernel = o.kernel == SPCONV_KERNEL_AUTO;
    if (o.kernel == SPCONV_KERNEL_AUTO) {
        p->kernel = pipe_ok ? SPCONV_KERNEL_PIPE : tiled_ok ? SPCONV_KERNEL_TILED : SPCONV_KERNEL_GENERIC;
        // the dense kernel at and above the measured break-even density,
        // which depends on how well the dense kernel's geometry fits the layer (judged at
        // a 32-image batch)
        if (dense_ok && density >= spconv::kDenseBreakEven) {
            const double eff = spconv::dense_expected_efficiency(*p, 32);
            p->dense = density >= (eff >= spconv::kDenseGoodGeometry ? spconv::kDenseBreakEven
                                                                       : spconv::kDenseBreakEvenWeak);
        }
    } else if (o.kernel == SPCONV_KERNEL_DENSE) {
        // fused / epilogue calls of a dense plan take AUTO's sparse kernel
        p->kernel = pipe_ok ? SPCONV_KERNEL_PIPE : tiled_ok ? SPCONV_KERNEL_TILED : SPCONV_KERNEL_GENERIC;
        p->dense = true;
    } else {
        p->kernel = o.kernel;
    }
    int R = o.rows_per_group;
    if (R == 0) {
        R = p->kernel == SPCONV_KERNEL_PIPE ? 4 : spconv::tiled_default_R(C, F, double(nnz) / (double(F) * ncol));
        // pipe: R = 2 (12 warps) once a row has >= 3.5 nonzeros per input channel
        // (density >= ~0.39): the per-channel window reload is then amortised and the
        // extra warps hide more dispatch latency.  Measured crossover 3.2-3.6 on the c2,
        // c4 and c5 shapes (profiles/r01_r_sweep.jsonl)
        if (p->kernel == SPCONV_KERNEL_PIPE && double(nnz) >= 3.5 * double(F) * double(C)) R = 2;
        // A/B switch for the pipe kernel's rows per group
        if (p->kernel == SPCONV_KERNEL_PIPE)
            if (const char *e = std::getenv("SPCONV_PIPE_R")) R = std::atoi(e);
    }
    if ((p->kernel == SPCONV_KERNEL_PIPE && R != 4 && R != 2) ||
        (p->kernel == SPCONV_KERNEL_TILED && R != 4 && R != 8)) {
        delete p;
        return SPCONV_ERR_UNSUPPORTED;
    }
    st = build_plan(p, h_rowptr, h_colidx, h_values, h_bias, R);
    if (!st && p->dense) {
        spconv::dense_geometry(*p, p->dense_geo);
        if (!p->dense_geo.ok) {
            if (o.kernel == SPCONV_KERNEL_DENSE) st = SPCONV_ERR_UNSUPPORTED;
            p->dense = false;
        } else {
            const std::vector<float> w = spconv::dense_weights(*p, p->dense_geo, h_rowptr, h_colidx, h_values);
            st = upload(&p->d_wdense, w.data(), w.size(), p->device_bytes);
        }
    }
    if (st) {
        free_plan(p);
        return st;
    }
    // the R = 2 alternate of an AUTO pipe plan (prefer_alt chooses per call)
    if (p->auto_kernel && p->kernel == SPCONV_KERNEL_PIPE && !p->dense && p->R == 4 &&
        density >= spconv::kAltMinDensity && !std::getenv("SPCONV_PIPE_R") && !std::getenv("SPCONV_NO_ALT")) {
        spconv_plan_s *q = new (std::nothrow) spconv_plan_s;
        if (q) {
            q->C = p->C; q->H = p->H; q->W = p->W; q->F = p->F; q->K = p->K; q->stride = p->stride;
            q->pad = p->pad; q->Ho = p->Ho; q->Wo = p->Wo; q->nnz = p->nnz; q->device = p->device;
            q->knobs = p->knobs;
            q->kernel = SPCONV_KERNEL_PIPE;
            q->density = density;
            if (build_plan(q, h_rowptr, h_colidx, h_values, h_bias, 2) == SPCONV_OK) {
                p->alt = q;
                p->device_bytes += q->device_bytes;
            } else {
                free_plan(q);
                cudaGetLastError();
            }
        }
    }
    *plan = p;
    return SPCONV_OK;
}

int spconv_create(spconv_plan_t *plan, int C, int H, int W, int F, int K, int stride, int pad,
                  const int32_t *rowptr, const int32_t *colidx, const float *values, int64_t nnz,
                  const float *bias, int device) {
    return spconv_create_ex(plan, C, H, W, F, K, stride, pad, rowptr, colidx, values, nnz, bias,
                            device, nullptr);
}

// AUTO's per-call choice between the pipe kernel and the generic one-thread-per-output
// kernel for SMALL calls (verdict r1 item 6).  Measured on B200 (profiles/r02/
// small_layers_*.jsonl): the pipe kernel's walk over the C input channels is latency
// bound when a call has few units (c4_95 N=1: 8 CTAs, 146 us; c2 N=1: 56 us), while the
// generic kernel's time is ~7 us + 1.2 ns per FMA (c1: 8 us, c2 N=1: 37 us).  Model:
//   generic_us = 7 + 1.2e-3 * N*F*Ho*Wo*(nnz/F) / 1000
//   pipe_us    = 5 + max(1, units/SMs) * C * (0.35 * P(a group has a tap in a channel)
//                                             + 0.075 * 9*R*density)
// and the generic kernel is taken when it is predicted 20% faster.  Both kernels obey
// the same FP32 contract, so the choice never changes a bit.
static bool small_call_prefers_generic(const Plan *p, int N, uintptr_t x) {
    if (!p->auto_kernel || p->kernel != SPCONV_KERNEL_PIPE || N <= 0) return false;
    const double d = double(p->nnz) / (double(p->F) * p->C * p->K * p->K);
    const double fma = double(N) * p->F * p->Ho * p->Wo * (double(p->nnz) / p->F);
    const double t_generic = 7.0 + 1.2e-6 * fma;
    spconv::PipeSchedule q;
    if (!spconv::pipe_schedule(*p, N, x, q, false)) return true;
    const double rounds = std::max(1.0, double(q.nunits) / double(spconv::sm_count_of_current_device()));
    const double p_nonempty = 1.0 - std::pow(1.0 - d, 9.0 * p->R);
    const double t_pipe = 5.0 + rounds * p->C * (0.35 * p_nonempty + 0.075 * 9.0 * p->R * d);
    return t_generic < 0.8 * t_pipe;
}

// Whether the pipelined kernel serves this call at all (its block epilogues need the
// default dispatcher; wide rows have a subset of instantiations -- pipe_schedule).
static bool pipe_serves(const Plan *p, int N, uintptr_t x, bool fused, int epi) {
    if (p->kernel != SPCONV_KERNEL_PIPE || (epi && p->pipe_dispatch == 1)) return false;
    spconv::PipeSchedule q;
    return spconv::pipe_schedule(*p, N, x, q, !fused, epi);
}

// Per call: the R = 2 alternate instead of the R = 4 plan?  A pipe launch takes about
// max(1, units / SMs) unit times (stream-K spreads a partial round), and an R = 2 unit
// (half the rows per warp, 12 warps per CTA instead of 8) takes r(density) of an R = 4
// unit: measured on B200 on the final kernel (profiles/r02/r_crossover_final.jsonl,
// ab_alt_r2*.jsonl) -- 0.96 at d = 0.05, 0.94 at 0.1, 0.79 at 0.2, 0.67 at 0.3.  c4_80
// (128 units at R = 4 leave 20 SMs idle; 176 at R = 2): 203.1 -> 190.6 us.
static double r2_unit_ratio(double d) {
    static const double xs[] = {0.05, 0.10, 0.20, 0.30, 0.40}, ys[] = {0.96, 0.94, 0.79, 0.67, 0.60};
    if (d <= xs[0]) return ys[0];
    for (int i = 1; i < 5; ++i)
        if (d <= xs[i]) return ys[i - 1] + (ys[i] - ys[i - 1]) * (d - xs[i - 1]) / (xs[i] - xs[i - 1]);
    return ys[4];
}

static bool prefer_alt(const Plan *p, int N, uintptr_t x, bool fused, int epi) {
    if (!p->alt || N <= 0) return false;
    spconv::PipeSchedule q4, q2;
    if (!spconv::pipe_schedule(*p, N, x, q4, !fused, epi) || !spconv::pipe_schedule(*p->alt, N, x, q2, !fused, epi))
        return false;
    const double sms = double(spconv::sm_count_of_current_device());
    // a stream-K launch adds a park, a resume and a partial unit per CTA: about 6
    // channel steps of a unit's C (c2 N=16: R = 2's 168 units on 148 SMs measured 5%
    // slower than R = 4's 112, while c4_80's 256-channel units gain 6%)
    auto rounds = [&](const spconv::PipeSchedule &q) {
        const double r = std::max(1.0, double(q.nunits) / sms);
        return q.sk ? r * (1.0 + 6.0 / double(p->C)) : r;
    };
    const double t4 = rounds(q4), t2 = rounds(q2) * r2_unit_ratio(p->density);
    return t2 < 0.97 * t4;
}

static int run(spconv_plan_t plan, int N, const float *x, float *y, int32_t *argmax, bool fused,
               void *stream, const float *res = nullptr, int flags = 0) {
    if (!plan) return SPCONV_ERR_NULLPTR;
    Plan *p = plan;
    if (flags & ~(SPCONV_EPI_RELU | SPCONV_EPI_RESIDUAL)) return SPCONV_ERR_UNSUPPORTED;
    if (N < 0) return SPCONV_ERR_SHAPE;
    if (fused && (p->Ho < 2 || p->Wo < 2)) return SPCONV_ERR_SHAPE;
    if (N == 0) return SPCONV_OK;
    if (!x || !y) return SPCONV_ERR_NULLPTR;
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
         reinterpret_cast<uintptr_t>(argmax)) & 3)
        return SPCONV_ERR_ALIGN;
    const size_t xbytes = size_t(N) * p->C * p->H * p->W * 4;
    const size_t ybytes = fused ? size_t(N) * p->F * (p->Ho / 2) * (p->Wo / 2) * 4
                                : size_t(N) * p->F * p->Ho * p->Wo * 4;
    if (overlap(x, xbytes, y, ybytes)) return SPCONV_ERR_ALIAS;
    if (argmax && (overlap(x, xbytes, argmax, ybytes) || overlap(y, ybytes, argmax, ybytes)))
        return SPCONV_ERR_ALIAS;
    if (flags & SPCONV_EPI_RESIDUAL) {
        if (!res) return SPCONV_ERR_NULLPTR;
        if (reinterpret_cast<uintptr_t>(res) & 3) return SPCONV_ERR_ALIGN;
        // the residual may be y itself (in-place accumulate) but not partially overlap it
        if (res != y && overlap(res, ybytes, y, ybytes)) return SPCONV_ERR_ALIAS;
    }
    int st;
    // device-pointer checks, cached per plan by pointer (a pointer once validated as this
    // device's memory is not re-queried; a caller that frees it and passes the same address
    // for host memory is outside the contract either way)
    auto checked = [&](const void *ptr) {
        if (p->cache.is_valid(ptr)) return int(SPCONV_OK);
        const int r = check_device_ptr(ptr, p->device);
        if (r == SPCONV_OK) p->cache.put_valid(ptr);
        return r;
    };
    if ((st = checked(x)) || (st = checked(y))) return st;
    if (argmax && (st = checked(argmax))) return st;
    if ((flags & SPCONV_EPI_RESIDUAL) && (st = checked(res))) return st;
    DeviceGuard guard(p->device);
    if (!guard.ok) return SPCONV_ERR_CUDA;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    const int epi = fused ? 0 : flags;
    if (p->dense)
        e = spconv::launch_dense(*p, N, x, y, argmax, fused, s, res, epi);
    else if (pipe_serves(p, N, reinterpret_cast<uintptr_t>(x), fused, epi) &&
             !small_call_prefers_generic(p, N, reinterpret_cast<uintptr_t>(x)))
        e = spconv::launch_pipe(prefer_alt(p, N, reinterpret_cast<uintptr_t>(x), fused, epi) ? *p->alt : *p, N, x, y,
                                argmax, fused, s, res, epi);
    else if (p->kernel == SPCONV_KERNEL_TILED && epi == 0)
        e = spconv::launch_tiled(*p, N, x, y, argmax, fused, s);
    else  // the generic kernel serves every epilogue the specialised kernel lacks
        e = fused ? spconv::launch_generic_fused(*p, N, x, y, argmax, s)
                  : spconv::launch_generic_conv(*p, N, x, y, s, res, epi);
    if (e == cudaSuccess && p->knobs.debug) { // SPCONV_DEBUG: report a fault at this call
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cap);
        if (cap == cudaStreamCaptureStatusNone) e = cudaStreamSynchronize(s); // (not inside a graph capture)
    }
    return e == cudaSuccess ? SPCONV_OK : cuda_fail(e);
}

int spconv_forward(spconv_plan_t plan, int N, const float *x, float *y, void *stream) {
    NvtxRange r("spconv_forward");
    return run(plan, N, x, y, nullptr, false, stream);
}

int spconv_fused_relu_maxpool(spconv_plan_t plan, int N, const float *x, float *y, int32_t *argmax,
                              void *stream) {
    NvtxRange r("spconv_fused_relu_maxpool");
    return run(plan, N, x, y, argmax, true, stream);
}

int spconv_resize_bilinear(int N, int C, const float *x, int Hin, int Win, float *y, int Hout, int Wout,
                           void *stream) {
    if (N < 0 || C < 1 || Hin < 1 || Win < 1 || Hout < 1 || Wout < 1) return SPCONV_ERR_SHAPE;
    if (N == 0) return SPCONV_OK;
    if (!x || !y) return SPCONV_ERR_NULLPTR;
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 3) return SPCONV_ERR_ALIGN;
    const size_t xb = size_t(N) * C * Hin * Win * 4, yb = size_t(N) * C * Hout * Wout * 4;
    if (overlap(x, xb, y, yb)) return SPCONV_ERR_ALIAS;
    cudaPointerAttributes ax, ay;
    if (cudaPointerGetAttributes(&ax, x) != cudaSuccess || cudaPointerGetAttributes(&ay, y) != cudaSuccess) {
        cudaGetLastError();
        return SPCONV_ERR_DEVICE;
    }
    if ((ax.type != cudaMemoryTypeDevice && ax.type != cudaMemoryTypeManaged) ||
        (ay.type != cudaMemoryTypeDevice && ay.type != cudaMemoryTypeManaged) || ax.device != ay.device)
        return SPCONV_ERR_DEVICE;
    DeviceGuard guard(ax.device);
    if (!guard.ok) return SPCONV_ERR_CUDA;
    cudaError_t e = spconv::launch_resize(x, y, int64_t(N) * C, Hin, Win, Hout, Wout, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? SPCONV_OK : cuda_fail(e);
}

int spconv_resize_fused_relu_maxpool(spconv_plan_t plan, int N, const float *x, int Hin, int Win, float *y,
                                     int32_t *argmax, void *stream) {
    if (!plan) return SPCONV_ERR_NULLPTR;
    Plan *p = plan;
    if (N < 0 || Hin < 1 || Win < 1) return SPCONV_ERR_SHAPE;
    if (p->Ho < 2 || p->Wo < 2) return SPCONV_ERR_SHAPE;
    if (N == 0) return SPCONV_OK;
    if (!x || !y) return SPCONV_ERR_NULLPTR;
    int st;
    if ((st = check_device_ptr(x, p->device))) return st;
    DeviceGuard guard(p->device);
    if (!guard.ok) return SPCONV_ERR_CUDA;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // the resized image lives in a stream-ordered workspace between the two launches
    spconv::keep_pool_cached();
    float *xr = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&xr), size_t(N) * p->C * p->H * p->W * 4, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return SPCONV_ERR_OOM;
    }
    st = spconv_resize_bilinear(N, p->C, x, Hin, Win, xr, p->H, p->W, stream);
    if (st == SPCONV_OK) st = run(plan, N, xr, y, argmax, true, stream);
    cudaFreeAsync(xr, s);
    return st;
}

int spconv_forward_ex(spconv_plan_t plan, int N, const float *x, const float *residual, float *y, int flags,
                      void *stream) {
    NvtxRange r("spconv_forward_ex");
    return run(plan, N, x, y, nullptr, false, stream, residual, flags);
}

int spconv_forward_host(spconv_plan_t plan, int N, const float *x_host, float *y_host, int fused,
                        int32_t *argmax_host) {
    NvtxRange nvtx("spconv_forward_host");
    if (!plan) return SPCONV_ERR_NULLPTR;
    Plan *p = plan;
    if (N < 0) return SPCONV_ERR_SHAPE;
    if (fused && (p->Ho < 2 || p->Wo < 2)) return SPCONV_ERR_SHAPE;
    if (N == 0) return SPCONV_OK;
    if (!x_host || !y_host) return SPCONV_ERR_NULLPTR;
    const size_t xn = size_t(N) * p->C * p->H * p->W;
    const size_t yn = fused ? size_t(N) * p->F * (p->Ho / 2) * (p->Wo / 2)
                            : size_t(N) * p->F * p->Ho * p->Wo;
    std::lock_guard<std::mutex> lock(p->host_mu);
    DeviceGuard guard(p->device);
    if (!guard.ok) return SPCONV_ERR_CUDA;
    if (!p->host_stream) {
        // three streams (copy in, compute, copy out) and per-chunk events, created once
        if (cudaStreamCreateWithFlags(&p->host_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&p->host_ostream, cudaStreamNonBlocking) != cudaSuccess)
            return SPCONV_ERR_CUDA;
        for (cudaStream_t &ks : p->host_kstream)
            if (cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking) != cudaSuccess) return SPCONV_ERR_CUDA;
        for (int i = 0; i < Plan::MAX_HOST_CHUNKS; ++i)
            if (cudaEventCreateWithFlags(&p->host_ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&p->host_ev_k[i], cudaEventDisableTiming) != cudaSuccess)
                return SPCONV_ERR_CUDA;
    }
    if (xn > p->xbuf_elems) {
        cudaFree(p->d_xbuf);
        p->d_xbuf = nullptr;
        p->xbuf_elems = 0;
        if (cudaMalloc(&p->d_xbuf, xn * 4) != cudaSuccess) { cudaGetLastError(); return SPCONV_ERR_OOM; }
        p->xbuf_elems = xn;
    }
    if (yn > p->ybuf_elems) {
        cudaFree(p->d_ybuf);
        cudaFree(p->d_abuf);
        p->d_ybuf = nullptr;
        p->d_abuf = nullptr;
        p->ybuf_elems = 0;
        if (cudaMalloc(&p->d_ybuf, yn * 4) != cudaSuccess || cudaMalloc(&p->d_abuf, yn * 4) != cudaSuccess) {
            cudaGetLastError();
            return SPCONV_ERR_OOM;
        }
        p->ybuf_elems = yn;
    }
    // Pipelined over contiguous image chunks (NCHW is batch-major, so a chunk is one
    // contiguous slice of x and y): the copy-in of chunk i+1 and the copy-out of
    // chunk i-1 overlap the forward of chunk i (PCIe is full duplex), so the call
    // costs about max(H2D, D2H) instead of H2D + forward + D2H.  A forward over a
    // few images fills only part of the GPU and is latency-bound, so the chunks'
    // forwards go round-robin to HOST_KSTREAMS streams and overlap each other too.
    // Each image is computed exactly as in one launch over the whole batch (images
    // are independent), so the result is bitwise the same.
    const size_t xper = xn / size_t(N), yper = yn / size_t(N);
    // >= 3 MiB of input per chunk, at most 8 (measured on c2: 8 chunks 0.74 ms, 1 chunk 1.04 ms,
    // 16 chunks 0.89 ms; the floor is the 0.54 ms of concurrent 25.7 MB copies each way)
    int nchunk = int(std::min<size_t>(8, (xn * 4) / (size_t(3) << 20)));
    if (const char *e = std::getenv("SPCONV_HOST_CHUNKS")) nchunk = std::atoi(e); // A/B tooling
    nchunk = std::max(1, std::min({nchunk, N, Plan::MAX_HOST_CHUNKS}));
    int32_t *dam = (fused && argmax_host) ? p->d_abuf : nullptr;
    // on an error after the first enqueue, drain the streams before returning so no
    // copy into or out of the caller's host buffers is still in flight
    auto drain = [&](int st) {
        cudaStreamSynchronize(p->host_stream);
        for (cudaStream_t ks : p->host_kstream) cudaStreamSynchronize(ks);
        cudaStreamSynchronize(p->host_ostream);
        cudaGetLastError();
        return st;
    };
    for (int i = 0, n0 = 0; i < nchunk; ++i) {
        const int n1 = int(int64_t(N) * (i + 1) / nchunk), nb = n1 - n0;
        const size_t xo = size_t(n0) * xper, yo = size_t(n0) * yper;
        cudaStream_t ks = p->host_kstream[i % Plan::HOST_KSTREAMS];
        if (cudaMemcpyAsync(p->d_xbuf + xo, x_host + xo, size_t(nb) * xper * 4, cudaMemcpyHostToDevice,
                            p->host_stream) != cudaSuccess ||
            cudaEventRecord(p->host_ev_in[i], p->host_stream) != cudaSuccess ||
            cudaStreamWaitEvent(ks, p->host_ev_in[i], 0) != cudaSuccess)
            return drain(SPCONV_ERR_CUDA);
        int st = run(plan, nb, p->d_xbuf + xo, p->d_ybuf + yo, dam ? dam + yo : nullptr, fused != 0, ks);
        if (st) return drain(st);
        if (cudaEventRecord(p->host_ev_k[i], ks) != cudaSuccess ||
            cudaStreamWaitEvent(p->host_ostream, p->host_ev_k[i], 0) != cudaSuccess ||
            cudaMemcpyAsync(y_host + yo, p->d_ybuf + yo, size_t(nb) * yper * 4, cudaMemcpyDeviceToHost,
                            p->host_ostream) != cudaSuccess)
            return drain(SPCONV_ERR_CUDA);
        if (dam && cudaMemcpyAsync(argmax_host + yo, dam + yo, size_t(nb) * yper * 4, cudaMemcpyDeviceToHost,
                                   p->host_ostream) != cudaSuccess)
            return drain(SPCONV_ERR_CUDA);
        n0 = n1;
    }
    // the copy-out stream waited on every forward, each of which waited on its copy-in
    if (cudaStreamSynchronize(p->host_ostream) != cudaSuccess) return SPCONV_ERR_CUDA;
    return SPCONV_OK;
}

int spconv_destroy(spconv_plan_t plan) {
    free_plan(plan);
    return SPCONV_OK;
}

int spconv_output_dims(spconv_plan_t plan, int N, int fused, int64_t dims[4]) {
    if (!plan || !dims) return SPCONV_ERR_NULLPTR;
    if (N < 0) return SPCONV_ERR_SHAPE;
    dims[0] = N;
    dims[1] = plan->F;
    dims[2] = fused ? plan->Ho / 2 : plan->Ho;
    dims[3] = fused ? plan->Wo / 2 : plan->Wo;
    return SPCONV_OK;
}

int spconv_launch_info(spconv_plan_t plan, int N, int fused, const float *x, spconv_launch_info_t *info) {
    if (!plan || !info) return SPCONV_ERR_NULLPTR;
    if (N < 0) return SPCONV_ERR_SHAPE;
    Plan *p = plan;
    *info = spconv_launch_info_t{};
    info->kernel = p->kernel;
    info->rows_per_group = p->R;
    info->launches = N > 0 ? 1 : 0;
    (void)fused;
    if (p->dense && N > 0) {
        const spconv::DenseGeometry &g = p->dense_geo;
        info->kernel = SPCONV_KERNEL_DENSE;
        info->rows_per_group = 8;
        const int64_t blocks = g.ipb > 1 ? (N + g.ipb - 1) / g.ipb : int64_t(N) * g.bpi;
        info->units = blocks * g.fsets;
        DeviceGuard guard(p->device);
        if (!guard.ok) return SPCONV_ERR_CUDA;
        info->grid = int(std::min<int64_t>(info->units, spconv::sm_count_of_current_device()));
        info->stream_k = spconv::dense_stream_k(*p, info->units, info->grid) ? 1 : 0;
        info->staging = (g.padded || (reinterpret_cast<uintptr_t>(x) & 15)) ? 1 : 0;
        info->channels_per_stage = g.cc;
        info->stages = g.nstage;
        info->launches = info->staging ? 2 : 1;
        return SPCONV_OK;
    }
    if (p->kernel == SPCONV_KERNEL_PIPE && N > 0) {
        DeviceGuard guard(p->device);
        if (!guard.ok) return SPCONV_ERR_CUDA;
        if (!pipe_serves(p, N, reinterpret_cast<uintptr_t>(x), fused != 0, 0) ||
            small_call_prefers_generic(p, N, reinterpret_cast<uintptr_t>(x))) {
            info->kernel = SPCONV_KERNEL_GENERIC;
            info->rows_per_group = 0;
            return SPCONV_OK;
        }
        if (prefer_alt(p, N, reinterpret_cast<uintptr_t>(x), fused != 0, 0)) {
            p = p->alt; // the call runs the R = 2 alternate
            info->rows_per_group = p->R;
        }
        spconv::PipeSchedule q;
        if (!spconv::pipe_schedule(*p, N, reinterpret_cast<uintptr_t>(x), q, !fused)) return SPCONV_ERR_UNSUPPORTED;
        info->grid = q.grid;
        info->stream_k = q.sk ? 1 : 0;
        info->units = q.nunits;
        info->band = q.g->band;
        info->staging = q.mode;
        info->channels_per_stage = q.g->cc;
        info->stages = q.g->nstage;
        info->launches = q.launches;
        info->tile_rows = q.g->T;
        info->sk_split = spconv::sk_table(*p, q, N, fused != 0, nullptr, nullptr) ? 1 : 0;
    }
    return SPCONV_OK;
}

int spconv_plan_info(spconv_plan_t plan, spconv_plan_info_t *info) {
    if (!plan || !info) return SPCONV_ERR_NULLPTR;
    const Plan *p = plan;
    std::memset(info, 0, sizeof(*info));
    info->C = p->C; info->H = p->H; info->W = p->W; info->F = p->F; info->K = p->K;
    info->stride = p->stride; info->pad = p->pad; info->Ho = p->Ho; info->Wo = p->Wo;
    info->nnz = p->nnz;
    info->device = p->device;
    info->kernel = p->dense ? SPCONV_KERNEL_DENSE : p->kernel; // the kernel of conv-only calls
    info->rows_per_group = p->R;
    info->num_groups = p->num_groups;
    info->device_bytes = p->device_bytes;
    // the pipelined / dense kernels need a padding pass first when TMA cannot stage the
    // caller's rows (W % 4 != 0); a misaligned base pointer adds it at run time
    info->launches_per_call = p->dense ? (p->dense_geo.padded ? 2 : 1)
                                       : (p->kernel == SPCONV_KERNEL_PIPE && !p->pipe_tma.ok) ? 2 : 1;
    return SPCONV_OK;
}

int spconv_debug_sk_split(const float *cost, int C, int gpc, int ngs, int num_groups, int cc, int64_t units,
                          int grid, int fused, int32_t *unit, uint16_t *ch) {
    if (!cost || !unit || !ch) return SPCONV_ERR_NULLPTR;
    if (C < 1 || gpc < 1 || gpc > spconv::kSkTabGpc || ngs < 1 || num_groups < 1 || num_groups > gpc * ngs ||
        cc < 1 || units < 1 || grid < 1 || grid > spconv::kSkTabCta)
        return SPCONV_ERR_SHAPE;
    std::vector<int32_t> u;
    std::vector<uint16_t> c;
    spconv::sk_split_core(cost, C, gpc, ngs, num_groups, cc, units, grid, fused != 0, u, c);
    if (u.empty()) return SPCONV_ERR_UNSUPPORTED; // no valid split: the launch uses the uniform one
    std::memcpy(unit, u.data(), u.size() * sizeof(int32_t));
    std::memcpy(ch, c.data(), c.size() * sizeof(uint16_t));
    return SPCONV_OK;
}

int spconv_debug_decoded(spconv_plan_t plan, int32_t *c, int32_t *dy, int32_t *dx) {
    if (!plan) return SPCONV_ERR_NULLPTR;
    const Plan *p = plan;
    if (p->nnz > 0 && (!c || !dy || !dx)) return SPCONV_ERR_NULLPTR;
    // Read back what was uploaded to the device, so the check covers the device copy.
    std::vector<uint32_t> taps(size_t(p->nnz));
    if (p->nnz) {
        DeviceGuard guard(p->device);
        if (cudaMemcpy(taps.data(), p->d_taps, taps.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
            return SPCONV_ERR_CUDA;
    }
    for (int64_t j = 0; j < p->nnz; ++j) {
        const uint32_t t = taps[size_t(j)];
        c[j] = int32_t(t >> 6);
        dy[j] = int32_t((t >> 3) & 7u) - p->pad;
        dx[j] = int32_t(t & 7u) - p->pad;
    }
    return SPCONV_OK;
}

} // extern "C"
