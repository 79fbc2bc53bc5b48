#!/usr/bin/env python
"""NEXT-1: sparsity sweep of the sparse kernel against dense
counterparts on the same B200, and the break-even density.

The paper's profitability result (P:L464-471 [Fig. breakeven]: "Above
certain density levels, a dense convolution implementation is more profitable
than the sparse counterpart ... break-even density level (43.5%)") was measured
on an i7 CPU against Tiramisu's own dense conv.  Here, for one layer shape, every
density d in the sweep is timed with:

* ``sparse``  — this library's sparse pipelined kernel (kernel="pipe") on a
  synthetic layer pruned to d;
* ``dense_own`` — this library's dense FP32 direct-conv kernel (kernel="dense",
  csrc/kernel_dense.cu: static FFMA2 code, no per-nonzero dispatch) on the fully
  dense layer -- its time does not depend on the density (SURVEY §8(f) "own dense
  FP32 direct conv");
* ``auto`` — what AUTO picks at d (the dense kernel at and above the break-even);
* ``cudnn_fp32`` — torch.nn.functional.conv2d in FP32 with TF32 disabled (library
  comparison, dense weights);
* ``cudnn_tf32`` — the same with TF32 tensor cores allowed (reported separately:
  a different precision).

Times are CUDA-event medians over rotating input sets larger than L2.  Output:
one JSON line per (density) plus a summary line with the break-even densities
(the density at which the sparse time reaches the dense time, linear
interpolation between sweep points; ``None`` if sparse stays faster).

    python scripts/breakeven.py [--shape c2|c4|c5] [--reps 30]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthgen  # noqa: E402
from paper_2005_04091_b200.breakeven import break_even_density  # noqa: E402

DENSITIES = [0.01, 0.02, 0.05, 0.10, 0.15, 0.20, 0.30, 0.40, 0.45, 0.50, 0.55, 0.60, 0.70, 0.80, 1.00]
L2 = 126 * 2**20


def _time(fn, reps, nsets):
    import torch
    for i in range(3):
        fn(i % nsets)
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(i % nsets)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    import torch
    from paper_2005_04091_b200 import SparseConv2d

    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="c2", choices=["c2", "c4", "c5"])
    ap.add_argument("--n", type=int, default=0, help="batch override (c5: 256 images is 1.6 GB)")
    ap.add_argument("--reps", type=int, default=30)
    args = ap.parse_args()
    base = synthgen.CONFIGS[{"c2": "c2", "c4": "c4_50", "c5": "c5"}[args.shape]]
    if args.n:
        base = base.with_batch(args.n)
    shape = (base.N, base.C, base.H, base.W)
    xh = synthgen.make_input(shape, synthgen.seed_of(base.k, 2))
    in_bytes = xh.nbytes
    out_bytes = base.N * base.F * base.Ho * base.Wo * 4
    nsets = max(2, math.ceil(2 * L2 / (in_bytes + out_bytes)))
    xs = [torch.from_numpy(xh).cuda() for _ in range(nsets)]
    ys = [torch.empty((base.N, base.F, base.Ho, base.Wo), device="cuda") for _ in range(nsets)]

    def sparse_time(d, kernel="pipe"):
        cfg = base.with_density(d)
        L = synthgen.make_layer(cfg, with_input=False)
        c = L.csr
        layer = SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, cfg.K, cfg.stride, cfg.pad, c.rowptr, c.colidx,
                             c.values, None, kernel=kernel)
        from paper_2005_04091_b200 import spconv
        ms = _time(lambda j: spconv.spconv_forward(layer.plan, cfg.N, xs[j].data_ptr(), ys[j].data_ptr(),
                                                   torch.cuda.current_stream().cuda_stream),
                   args.reps, nsets)
        kern = layer.info["kernel"]
        layer.close()
        return ms, cfg.nnz, kern

    dense_flops = 2 * base.F * base.C * 9 * base.N * base.Ho * base.Wo
    dense_ms, _, _ = sparse_time(1.0, "dense")
    w = torch.from_numpy(synthgen.make_input((base.F, base.C, 3, 3), 12345)).cuda()

    def cudnn(tf32):
        torch.backends.cudnn.allow_tf32 = tf32
        torch.backends.cuda.matmul.allow_tf32 = tf32
        return _time(lambda j: torch.nn.functional.conv2d(xs[j], w, padding=1), args.reps, nsets)

    cudnn_fp32 = cudnn(False)
    cudnn_tf32 = cudnn(True)
    torch.backends.cudnn.allow_tf32 = False
    rows = []
    for d in DENSITIES:
        ms, nnz, kern = sparse_time(d)
        auto_ms, _, auto_k = sparse_time(d, "auto")
        useful = 2 * nnz * base.N * base.Ho * base.Wo
        names = {1: "generic", 2: "tiled", 3: "pipe", 4: "dense"}
        row = {"shape": args.shape, "density": d, "nnz": nnz, "kernel": names[kern],
               "sparse_ms": round(ms, 5), "sparse_useful_tflops": round(useful / ms / 1e9, 3),
               "auto_kernel": names[auto_k], "auto_ms": round(auto_ms, 5),
               "dense_own_ms": round(dense_ms, 5), "dense_own_tflops": round(dense_flops / dense_ms / 1e9, 3),
               "cudnn_fp32_ms": round(cudnn_fp32, 5),
               "cudnn_tf32_ms": round(cudnn_tf32, 5),
               "speedup_vs_cudnn_fp32": round(cudnn_fp32 / ms, 3),
               "cudnn_fp32_tflops": round(dense_flops / cudnn_fp32 / 1e9, 3)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    dens = [r["density"] for r in rows]
    sp = [r["sparse_ms"] for r in rows]
    summary = {"shape": args.shape, "config": f"N={base.N} C=F={base.C} H=W={base.H} K=3 pad=1",
               "dense_own_tflops": round(dense_flops / dense_ms / 1e9, 3),
               "break_even_vs_dense_own": break_even_density(dens, sp, dense_ms),
               "break_even_vs_cudnn_fp32": break_even_density(dens, sp, cudnn_fp32),
               "break_even_vs_cudnn_tf32": break_even_density(dens, sp, cudnn_tf32),
               "paper": "43.5% density on an i7-6700HQ vs Tiramisu dense (P:L505), context only"}
    print(json.dumps({"summary": summary}), flush=True)


if __name__ == "__main__":
    main()
