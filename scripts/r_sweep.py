#!/usr/bin/env python
"""Rows per group of the pipelined kernel: R = 4 (8 warps) vs R = 2 (11-12 warps)
over a density sweep on the c2 (64 ch, 56x56, N=32), c4 (256 ch, 14x14, N=64) and
c5 (128 ch, 112x112, N=16) shapes.  CUDA-event medians over rotating input sets
larger than L2 (scripts/breakeven.py's timer).  One JSON line per (shape, density).

    python scripts/r_sweep.py [--reps 30]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import synthgen  # noqa: E402
from breakeven import _time, L2  # noqa: E402

DENSITIES = [0.05, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.8, 1.0]


def main():
    import torch
    from paper_2005_04091_b200 import SparseConv2d, spconv

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--shapes", default="c2,c4_50,c5")
    args = ap.parse_args()
    for name in args.shapes.split(","):
        base = synthgen.CONFIGS[name]
        if name == "c5":
            base = base.with_batch(16)
        xh = synthgen.make_input((base.N, base.C, base.H, base.W), synthgen.seed_of(base.k, 2))
        out_bytes = base.N * base.F * base.Ho * base.Wo * 4
        nsets = max(2, math.ceil(2 * L2 / (xh.nbytes + out_bytes)))
        xs = [torch.from_numpy(xh).cuda() for _ in range(nsets)]
        ys = [torch.empty((base.N, base.F, base.Ho, base.Wo), device="cuda") for _ in range(nsets)]
        for d in DENSITIES:
            cfg = base.with_density(d)
            c = synthgen.make_layer(cfg, with_input=False).csr
            row = {"shape": name, "N": cfg.N, "C": cfg.C, "HW": cfg.H, "density": d,
                   "nnz_per_row_channel": round(cfg.nnz / (cfg.F * cfg.C), 3)}
            for R in (4, 2):
                layer = SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, cfg.K, cfg.stride, cfg.pad, c.rowptr, c.colidx,
                                     c.values, None, kernel="pipe", rows_per_group=R)
                ms = _time(lambda j: spconv.spconv_forward(layer.plan, cfg.N, xs[j].data_ptr(), ys[j].data_ptr(),
                                                           torch.cuda.current_stream().cuda_stream),
                           args.reps, nsets)
                layer.close()
                row[f"R{R}_ms"] = round(ms, 5)
                row[f"R{R}_tflops"] = round(2 * cfg.nnz * cfg.N * cfg.Ho * cfg.Wo / ms / 1e9, 3)
            row["R2_over_R4"] = round(row["R4_ms"] / row["R2_ms"], 3)
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
