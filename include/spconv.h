/*
 * spconv.h — C-ABI of libspconv.so: CSR sparse direct convolution on B200
 * (sm_100a), optionally fused with bias + ReLU + 2x2 max-pool.
 *
 * The operation (arXiv 2005.04091, /root/reference/PAPER.md):
 *   * CSR filters (¶"Sparse Convolution with CSR"): the
 *     (F, C, K, K) weight tensor is flattened to (F, C*K*K) and its rows are
 *     compressed.  colidx[j] = (c*K + ky)*K + kx (reading G1),
 *     strictly ascending within a row.
 *   * Convolution (DSL listing; CSR loop L393-401):
 *       y[n][f][oy][ox] = bias[f] + sum_{j in row f, ascending}
 *                         values[j] * X(n, c_j, oy*stride + ky_j - pad,
 *                                            ox*stride + kx_j - pad)
 *     X = input inside [0,H)x[0,W), 0 outside (zero padding, reading G6).
 *     Ho = (H + 2*pad - K)/stride + 1, Wo = (W + 2*pad - K)/stride + 1.
 *     Arithmetic contract (reading G7): per output, FP32 fused multiply-add
 *     in ascending colidx order starting from +0 (padding taps contribute
 *     exactly nothing), then one FP32 add of the bias.  Results are
 *     bit-identical to the FP32-ordered oracle.
 *   * Fused block ("Conv-Relu-Maxpool"): r = ReLU(conv),
 *     ReLU(v) = v > 0 ? v : +0; pooled[py][px] = max over the 2x2 window at
 *     (2py, 2px), stride 2, floor (odd trailing row/column dropped, G9);
 *     argmax = flat index (2py+dy)*Wo + (2px+dx) of the FIRST window element
 *     in row-major order attaining the max (strict '>', G10) — the
 *     convention of torch.nn.functional.max_pool2d(return_indices=True).
 *
 * Layouts: activations are contiguous NCHW float32; outputs NFHoWo (conv) or
 * N F (Ho/2) (Wo/2) (fused).  All sizes are element counts.
 *
 * Ownership: rowptr/colidx/values/bias are deep-copied by spconv_create and
 * may be host OR device pointers (classified with cudaPointerGetAttributes);
 * the caller may free them afterwards.  x, y and argmax of the device entry
 * points are caller-owned DEVICE buffers on the plan's device, 4-byte
 * aligned; y must not overlap x; y is overwritten (never accumulated into).
 * A plan is immutable after creation and may be used concurrently on
 * different streams.
 *
 * Errors: every argument is checked before any launch; on error nothing is
 * written and a negative SPCONV_ERR_* code is returned.  Device entry points
 * are asynchronous on `stream` (a cudaStream_t passed as void*, NULL = the
 * legacy default stream); launch failures return SPCONV_ERR_CUDA.  There is
 * no CPU fallback: host pointers for x/y return SPCONV_ERR_DEVICE.
 */
#ifndef SPCONV_H_
#define SPCONV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPCONV_ABI_VERSION 1

enum {
    SPCONV_OK = 0,
    SPCONV_ERR_NULLPTR = -1,     /* a required pointer is NULL                     */
    SPCONV_ERR_SHAPE = -2,       /* sizes < 1, Ho/Wo < 1, N < 0, nnz mismatch      */
    SPCONV_ERR_CSR = -3,         /* rowptr/colidx malformed, unsorted, duplicate,
                                    out of range, or a non-finite value/bias       */
    SPCONV_ERR_UNSUPPORTED = -4, /* K > 8, stride > 8, pad > 16, sizes > int32     */
    SPCONV_ERR_ALIGN = -5,       /* x/y/argmax not 4-byte aligned                  */
    SPCONV_ERR_DEVICE = -6,      /* pointer not device memory of the plan's device */
    SPCONV_ERR_CUDA = -7,        /* a CUDA runtime call or launch failed           */
    SPCONV_ERR_OOM = -8,         /* device or host allocation failed               */
    SPCONV_ERR_ALIAS = -9,       /* y (or argmax) overlaps x                        */
    SPCONV_ERR_INTERNAL = -10    /* SPCONV_DEBUG=1 self-check of a plan failed       */
};

/* Environment (read once, when a plan is created): SPCONV_DEBUG=1 turns on extra
 * validation -- create rebuilds every output channel's (colidx, value) sequence from
 * the generated tap streams and compares it with the CSR (SPCONV_ERR_INTERNAL on a
 * mismatch); every device entry point synchronises its stream and reports a launch or
 * execution fault as SPCONV_ERR_CUDA at the call that caused it. */

/* Kernel selection (spconv_create_ex).  AUTO picks the dense kernel for K = 3,
 * stride 1, pad 1 layers at or above the break-even density, else the pipelined
 * kernel when the shape is supported by it (K = 3, stride 1, pad 1; rows wider than
 * 125 outputs in column blocks),
 * else the register-tiled v1 kernel when its staging fits shared memory, else the
 * generic kernel.
 * All are CUDA kernels; all obey the same arithmetic contract. */
enum {
    SPCONV_KERNEL_AUTO = 0,
    SPCONV_KERNEL_GENERIC = 1,   /* one thread per output; any supported shape    */
    SPCONV_KERNEL_TILED = 2,     /* v1: row-grouped register tiles, cp.async      */
    SPCONV_KERNEL_PIPE = 3,      /* v2: warp-specialised TMA pipeline, FFMA2      */
    SPCONV_KERNEL_DENSE = 4      /* dense FP32 direct conv of the densified filters
                                    (conv-only calls; fused / epilogue calls use PIPE).
                                    Bitwise equal to the others: a zero tap is an
                                    exact no-op of the FP32 contract.  AUTO picks it
                                    for layers denser than the measured break-even
                                    (DESIGN.md NEXT-1) */
};

typedef struct spconv_plan_s *spconv_plan_t;

typedef struct {
    int kernel;       /* SPCONV_KERNEL_*                                         */
    int rows_per_group; /* output channels per register tile (0 = auto): tiled 4|8, pipe 4|2 */
    int reserved[6];  /* must be zero                                           */
} spconv_options_t;

typedef struct {
    int C, H, W, F, K, stride, pad, Ho, Wo;
    int64_t nnz;
    int device;
    int kernel;           /* kernel a conv-only call launches (SPCONV_KERNEL_*)  */
    int rows_per_group;   /* tiled: R                                            */
    int num_groups;       /* tiled: ceil(F / R)                                  */
    int64_t device_bytes; /* device memory held by the plan                      */
    int launches_per_call;/* kernel launches per forward / fused call            */
} spconv_plan_info_t;

/* Create a plan on CUDA device `device` (PAPER.md L391 CSR; SURVEY.md §8(a)
 * a1-a3): validates the CSR, decodes colidx -> (c, ky, kx), groups output
 * channels by nnz for the tiled kernel and uploads everything.  `bias` may be
 * NULL (== 0).  nnz == 0 is legal (y = bias).  On success *plan is set. */
int spconv_create(spconv_plan_t *plan, int C, int H, int W, int F, int K, int stride,
                  int pad, const int32_t *rowptr /* F+1 */, const int32_t *colidx /* nnz */,
                  const float *values /* nnz */, int64_t nnz, const float *bias /* F|NULL */,
                  int device);

/* Same, with options (opts may be NULL == defaults). */
int spconv_create_ex(spconv_plan_t *plan, int C, int H, int W, int F, int K, int stride,
                     int pad, const int32_t *rowptr, const int32_t *colidx,
                     const float *values, int64_t nnz, const float *bias, int device,
                     const spconv_options_t *opts);

/* y[N][F][Ho][Wo] = conv(x) + bias.  x: device float[N*C*H*W]; y: device
 * float[N*F*Ho*Wo].  N == 0 is a no-op.  Asynchronous on `stream`. */
int spconv_forward(spconv_plan_t plan, int N, const float *x, float *y, void *stream);

/* Epilogue flags of spconv_forward_ex (VGG / ResNet
 * blocks chain conv layers with fused ReLU and residual add; PAPER.md L503,
 * L514: operator fusion). */
enum { SPCONV_EPI_RELU = 1, SPCONV_EPI_RESIDUAL = 2 };

/* y = [ReLU]( (conv(x) + bias) [+ residual] ) elementwise over N*F*Ho*Wo, the
 * two additions in that order, each one FP32 add (RN); ReLU(v) = v > 0 ? v : +0.
 * residual: device float[N*F*Ho*Wo], required iff flags has SPCONV_EPI_RESIDUAL;
 * it may be y itself (in-place accumulate) but must not partially overlap y.
 * flags == 0 is spconv_forward.  Errors and asynchrony as spconv_forward;
 * unknown flag bits return SPCONV_ERR_UNSUPPORTED. */
int spconv_forward_ex(spconv_plan_t plan, int N, const float *x, const float *residual, float *y,
                      int flags, void *stream);

/* Bilinear resize ("preceded by an image
 * resizing step"; the paper does not define it — DESIGN.md reading R2):
 * half-pixel centres (align_corners = False), source coordinate clamped below at
 * 0, neighbours clamped to the image, plain FP32 in the order
 *   s = (o + 0.5) * (in / out) - 0.5;  v = hy*(hx*v00 + lx*v01) + ly*(hx*v10 + lx*v11).
 * x: device float[N][C][Hin][Win]; y: device float[N][C][Hout][Wout] (not
 * overlapping x).  Asynchronous on `stream`. */
int spconv_resize_bilinear(int N, int C, const float *x, int Hin, int Win, float *y, int Hout, int Wout,
                           void *stream);

/* The Resize-Conv-Relu-Maxpool block: x [N][C][Hin][Win]
 * is resized to the plan's H x W, then y / argmax as spconv_fused_relu_maxpool.
 * The resized image is kept in a stream-ordered device workspace between the
 * two launches (the conv never re-reads x). */
int spconv_resize_fused_relu_maxpool(spconv_plan_t plan, int N, const float *x, int Hin, int Win,
                                     float *y, int32_t *argmax, void *stream);

/* y[N][F][Ho/2][Wo/2] = maxpool2x2(ReLU(conv(x) + bias)); argmax (device
 * int32, same shape, may be NULL) = first-max flat index within each (n,f)
 * conv-output plane.  Requires Ho >= 2 and Wo >= 2 (else SPCONV_ERR_SHAPE).
 * The conv output is never materialised (fusion). */
int spconv_fused_relu_maxpool(spconv_plan_t plan, int N, const float *x, float *y,
                              int32_t *argmax, void *stream);

/* End-to-end convenience entry point with HOST buffers: copies x_host to the
 * device, runs the forward (fused != 0: the fused block, argmax_host may be
 * NULL), copies the result back and synchronises.  Device staging buffers are
 * owned by the plan and grown on demand (serialised by an internal lock).
 * The batch is split into up to 8 contiguous image chunks (>= 3 MiB of input
 * each) pipelined over plan-owned streams, so the copy-in of chunk i+1 and
 * the copy-out of chunk i-1 overlap the forward of chunk i; the result is bitwise
 * that of one device-side call (images are independent).
 * Host buffers may be pageable or pinned (pinned is needed for the overlap). */
int spconv_forward_host(spconv_plan_t plan, int N, const float *x_host, float *y_host,
                        int fused, int32_t *argmax_host);

/* Frees the plan and its device memory.  NULL is accepted (no-op). */
int spconv_destroy(spconv_plan_t plan);

/* dims = {N, F, Ho, Wo} (fused == 0) or {N, F, Ho/2, Wo/2} (fused != 0). */
int spconv_output_dims(spconv_plan_t plan, int N, int fused, int64_t dims[4]);

int spconv_plan_info(spconv_plan_t plan, spconv_plan_info_t *info);

/* The launch schedule of one forward of N images (fused != 0: the fused block)
 * with input x (its alignment selects the staging path; NULL = 16-byte aligned).
 * Describes exactly what spconv_forward / spconv_fused_relu_maxpool would launch
 * (same decision code); the parity tests assert on it (stream-K really engaged,
 * band units, staging path).  The pipe-only fields are 0 for other kernels. */
typedef struct {
    int kernel;             /* SPCONV_KERNEL_* the call launches                   */
    int rows_per_group;     /* output channels per register tile                  */
    int grid;               /* pipe: persistent CTAs (<= SM count)                */
    int stream_k;           /* pipe: 1 = ordered stream-K split of the units      */
    int64_t units;          /* pipe: (pixel block, group set) work units          */
    int band;               /* pipe: 1 = units are one-tile-row bands             */
    int staging;            /* pipe: 0 TMA on x, 1 TMA on a padded copy, 2 cp.async */
    int channels_per_stage; /* pipe: input channels per pipeline stage            */
    int stages;             /* pipe: pipeline depth (shared-memory ring)          */
    int launches;           /* kernel launches per call                           */
    int tile_rows;          /* pipe: output rows per thread tile (8, or 7 for conv-only
                               calls on heights that are multiples of 7)            */
    int sk_split;           /* pipe, stream-K: 1 = per-warp cost-balanced split points
                               (each warp's range walks the same cost), 0 = uniform
                               channel split (SPCONV_PIPE_SK_SPLIT=uniform)         */
    int reserved[5];
} spconv_launch_info_t;
int spconv_launch_info(spconv_plan_t plan, int N, int fused, const float *x, spconv_launch_info_t *info);

/* Static string for a status code (never NULL). */
const char *spconv_status_string(int status);

int spconv_abi_version(void);

/* Static description of the last CUDA runtime error an entry point of this
 * library returned SPCONV_ERR_CUDA for on the calling thread (never NULL). */
const char *spconv_last_cuda_error(void);

/* Test-only: the decoded taps held by the plan, host outputs of nnz each:
 * c[j], dy[j] = ky_j - pad, dx[j] = kx_j - pad. */
int spconv_debug_decoded(spconv_plan_t plan, int32_t *c, int32_t *dy, int32_t *dx);

/* Test-only, host code (no GPU): the per-warp stream-K split points the pipe kernel's
 * launch would use (DESIGN.md §6 "Per-warp split points") for units work units of C
 * channel steps on grid CTAs of gpc warps, from cost[(gset*gpc + warp)*C + c] = the
 * walk cost of that warp's row group in channel c (ngs group sets, num_groups groups;
 * cc channels per pipeline stage; fused selects the epilogue cost).  Outputs unit[grid+1]
 * (the unit of boundary b) and ch[(grid+1)*gpc] (warp w's split channel in it).
 * SPCONV_ERR_SHAPE on bad sizes (grid <= 160, gpc <= 12); SPCONV_ERR_UNSUPPORTED when no
 * valid split exists (the launch then uses the uniform channel split). */
int spconv_debug_sk_split(const float *cost, int C, int gpc, int ngs, int num_groups, int cc, int64_t units,
                          int grid, int fused, int32_t *unit, uint16_t *ch);

#ifdef __cplusplus
}
#endif
#endif /* SPCONV_H_ */
