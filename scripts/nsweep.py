#!/usr/bin/env python
"""Batch-size sweep of one layer shape: kernel time vs N (work units per persistent
CTA), with ordered stream-K on and off (SPCONV_PIPE_SK).  Diagnoses the unit
quantisation of the persistent pipe kernel.

    python scripts/nsweep.py [--config c2] [--ns 8,16,...] [--reps 50]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402


def main():
    import torch
    from paper_2005_04091_b200 import SparseConv2d
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--ns", default="8,16,18,19,24,32,37,40,48,64")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--sk", default="0,1")
    ap.add_argument("--inner", type=int, default=10)
    a = ap.parse_args()
    base = synthgen.CONFIGS[a.config]
    Lw = synthgen.make_layer(base, with_input=False)
    c = Lw.csr
    layer = SparseConv2d(base.C, base.H, base.W, base.F, 3, 1, 1, c.rowptr, c.colidx, c.values,
                         synthgen.make_bias(base.F, 11))
    ns = [int(v) for v in a.ns.split(",")]
    xs_all = torch.from_numpy(synthgen.make_input((max(ns), base.C, base.H, base.W), 5)).cuda()
    for n in ns:
        x = xs_all[:n].contiguous()
        for sk in a.sk.split(","):
            os.environ["SPCONV_PIPE_SK"] = sk
            fn = layer.fused_relu_maxpool if base.fused else layer
            for _ in range(5):
                fn(x)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                fn(x)  # queue ahead so the events bracket device time only
                e0.record()
                for _ in range(a.inner):
                    fn(x)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) / a.inner)
            ms = statistics.median(ts)
            flops = 2.0 * c.nnz * n * base.H * base.W
            print(json.dumps({"config": a.config, "N": n, "sk": sk, "ms": round(ms, 5),
                              "gflops": round(flops / ms / 1e6, 1)}), flush=True)
    layer.close()


if __name__ == "__main__":
    main()
