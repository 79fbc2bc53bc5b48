"""A/B timing of library builds (SPCONV_LIB) and env knobs on BASELINE.json configs.

    python scripts/ab_time.py --libs ab/a.so,ab/b.so --configs c2,c3 [--rounds 3] [--env K=V ...]
    python scripts/ab_time.py --density-sweep c2 --densities 0.01,0.05,0.1,0.2,0.3

Each (lib, config) runs in its own process (a library is loaded once per process),
interleaved over --rounds so that clock drift hits every variant alike.  Per run:
plan built once, 10 warm-ups, then `reps` groups of back-to-back launches between two
events (inputs rotate over sets larger than the L2); reports the median group's
us/launch and useful TFLOP/s.  Prints one JSON line per run.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(cfg_name, density, iters, reps, kernel, rows, batch=0):
    import numpy as np
    import torch

    import synthgen
    from paper_2005_04091_b200 import spconv
    if cfg_name.startswith("custom:"):  # custom:N,C,H,W,F,density (K=3 pad 1)
        n_, c_, h_, w_, f_, d_ = cfg_name.split(":", 1)[1].split(",")
        cfg = synthgen.LayerConfig(6, "custom", int(n_), int(c_), int(h_), int(w_), int(f_), 3, 1, 1, float(d_),
                                   False, False)
    else:
        cfg = synthgen.CONFIGS[cfg_name]
    if density:
        cfg = cfg.with_density(density)
    if batch:
        cfg = cfg.with_batch(batch)
    L = synthgen.make_layer(cfg)
    layer = spconv.SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, cfg.K, cfg.stride, cfg.pad, L.csr.rowptr,
                                L.csr.colidx, L.csr.values, L.bias, kernel=kernel, rows_per_group=rows)
    oshape = layer.output_shape(cfg.N, cfg.fused)
    per = L.x.nbytes + int(np.prod(oshape)) * 8
    nsets = max(2, math.ceil(3 * 126 * 2**20 / per))
    xs = [torch.from_numpy(L.x).cuda() for _ in range(nsets)]
    ys = [torch.empty(oshape, device="cuda") for _ in range(nsets)]
    am = [torch.empty(oshape, dtype=torch.int32, device="cuda") for _ in range(nsets)] if cfg.fused else None
    sh = torch.cuda.current_stream().cuda_stream

    def step(i):
        j = i % nsets
        if cfg.fused:
            spconv.spconv_fused_relu_maxpool(layer.plan, cfg.N, xs[j].data_ptr(), ys[j].data_ptr(),
                                             am[j].data_ptr(), sh)
        else:
            spconv.spconv_forward(layer.plan, cfg.N, xs[j].data_ptr(), ys[j].data_ptr(), sh)

    for i in range(10):
        step(i)
    torch.cuda.synchronize()
    res = []
    k = 0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            step(k)
            k += 1
        b.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / iters)
    ms = statistics.median(res)
    info = layer.info
    out = {"lib": os.environ.get("SPCONV_LIB", "default"), "config": cfg_name, "density": cfg.density,
           "N": cfg.N, "kernel_req": kernel,
           "us": round(ms * 1e3, 3), "tflops": round(cfg.useful_flops / ms / 1e9, 3),
           "min_us": round(min(res) * 1e3, 3), "R": int(info["rows_per_group"]),
           "kernel": int(info["kernel"]),
           "env": {k: v for k, v in os.environ.items() if k.startswith("SPCONV_") and k != "SPCONV_LIB"}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", default="")
    ap.add_argument("--configs", default="c2")
    ap.add_argument("--densities", default="")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--envs", default="", help="';'-separated env sets, each 'K=V,K=V' (A/B knobs)")
    ap.add_argument("--batches", default="", help="comma-separated batch overrides")
    ap.add_argument("--kernels", default="", help="comma-separated kernels to compare (overrides --kernel)")
    ap.add_argument("--child", nargs=2)
    ap.add_argument("--batch", type=int, default=0)
    args = ap.parse_args()
    if args.child:
        child(args.child[0], float(args.child[1]), args.iters, args.reps, args.kernel, args.rows, args.batch)
        return
    libs = [os.path.abspath(x) for x in args.libs.split(",") if x] or [""]
    envs = [dict(kv.split("=", 1) for kv in e.split(",") if kv) for e in args.envs.split(";")] if args.envs else [{}]
    dens = [float(d) for d in args.densities.split(",") if d] or [0.0]
    batches = [int(b) for b in args.batches.split(",") if b] or [0]
    kernels = [k for k in args.kernels.split(",") if k] or [args.kernel]
    for _ in range(args.rounds):
        for c in args.configs.split(";" if ";" in args.configs or args.configs.startswith("custom:") else ","):
            for d in dens:
                for bt in batches:
                    for kern in kernels:
                        for lib in libs:
                            for e in envs:
                                env = dict(os.environ, **e)
                                if lib:
                                    env["SPCONV_LIB"] = lib
                                subprocess.run([sys.executable, __file__, "--child", c, str(d), "--iters",
                                                str(args.iters), "--reps", str(args.reps), "--kernel", kern,
                                                "--rows", str(args.rows), "--batch", str(bt)], env=env, timeout=600)


if __name__ == "__main__":
    main()
