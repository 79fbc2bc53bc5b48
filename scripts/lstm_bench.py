#!/usr/bin/env python
"""NEXT-4: the sparse multilayer LSTM at the paper's sizes
(4 layers, 100 time steps, 1024 hidden units, 15% uniformly
distributed density; D = 1024 inputs, batch B), wavefront vs sequential schedule.

Prints one JSON line per schedule: ms per forward (CUDA-event median), useful
GFLOP/s (2 * nnz * B per cell, summed over the L*T cells), kernel launches, and the
max |error| against the float64 oracle on a sample of batch columns.

    python scripts/lstm_bench.py [--batch 64] [--reps 20]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthgen  # noqa: E402


def main():
    import torch
    from paper_2005_04091_b200.lstm import SEQUENTIAL, WAVEFRONT, SparseLSTM
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--T", type=int, default=100)
    a = ap.parse_args()
    L, D, H, d, T, B = 4, 1024, 1024, 0.15, a.T, a.batch
    layers, x = synthgen.make_lstm(L, D, H, d, T, B)
    nnz = sum(len(l[1]) for l in layers)
    flops = 2 * nnz * B * T
    net = SparseLSTM(D, H, layers)
    xt = torch.from_numpy(x).cuda()
    sample = [0, B // 2, B - 1]
    import oracle
    ref = oracle.lstm_f64(np.ascontiguousarray(x[:, sample, :]), layers, H)
    for name, sch in (("wavefront", WAVEFRONT), ("sequential", SEQUENTIAL)):
        out = net(xt, sch)
        for _ in range(2):
            net(xt, sch, out=out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            net(xt, sch, out=out)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        err = float(np.abs(out.cpu().numpy()[:, sample, :] - ref).max())
        print(json.dumps({"lstm": name, "L": L, "D": D, "H": H, "T": T, "B": B, "density": d, "nnz": nnz,
                          "ms": round(ms, 3), "useful_gflops": round(flops / ms / 1e6, 1),
                          "sequences_per_s": round(B / ms * 1e3, 1), "launches": net.launches(T, sch),
                          "max_abs_err_vs_f64_oracle": err,
                          "data": "synthetic CSR at 15% density (PAPER.md L510), values scaled 1/sqrt(row nnz)"}),
              flush=True)
    net.close()


if __name__ == "__main__":
    main()
