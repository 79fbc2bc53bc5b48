#!/usr/bin/env python
"""NEXT-3: throughput of whole sparse blocks on one B200.

* ResNet-20 "block 10" shape: the basic block of layers 9-10 (Table 1, PAPER.md
  L364-370: densities 20.3% and 16.1%), 32 channels at 16x16 (CIFAR), N=256,
  identity shortcut, ReLU and the residual add fused into the conv epilogues.
* VGG-16 "block 10" shape: conv4_1..conv4_3 (densities 24.2%, 5.8%, 1.0%), 256 ->
  512 -> 512 channels at 28x28 (ImageNet), N=16, ReLU fused, max-pool fused into
  the last conv.

Synthetic weights/inputs (synthgen); CUDA-event median over rotating input sets.
Prints one JSON line per block: useful GFLOP/s (sum over layers of 2*nnz*N*Ho*Wo),
images/s, ms per block, kernel launches per block.

    python scripts/blocks_bench.py [--reps 50]
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

import synthgen  # noqa: E402
from paper_2005_04091_b200.blocks import (RESNET20_BLOCK10, VGG16_BLOCK10, ResNetBasicBlock,  # noqa: E402
                                          VGGBlock, make_layer)

L2 = 126 * 2**20


def run(name, spec, N, reps, kind):
    import torch
    H, W = spec["H"], spec["W"]
    layers, flops = [], 0
    for i, s in enumerate(spec["layers"]):
        csr = synthgen.make_csr(s.F, s.C, 3, s.density, 7000 + 10 * i, 7001 + 10 * i)
        bias = synthgen.make_bias(s.F, 7002 + 10 * i)
        layers.append(make_layer(s, H, W, csr, bias))
        flops += 2 * csr.nnz * N * H * W
    blk = ResNetBasicBlock(*layers) if kind == "resnet" else VGGBlock(layers)
    C0 = spec["layers"][0].C
    x_bytes = N * C0 * H * W * 4
    nsets = max(2, math.ceil(2 * L2 / x_bytes))
    xs = [torch.from_numpy(synthgen.make_input((N, C0, H, W), 7100 + k)).cuda() for k in range(min(nsets, 4))]
    nsets = len(xs)
    for i in range(3):
        blk(xs[i % nsets])
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        blk(xs[i % nsets])
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    launches = sum(int(layer.info["launches_per_call"]) for layer in layers)
    line = {"block": name, "N": N, "H": H, "W": W,
            "layers": [{"C": s.C, "F": s.F, "density": s.density} for s in spec["layers"]],
            "ms": round(ms, 4), "images_per_s": round(N / ms * 1e3, 1),
            "useful_gflops": round(flops / ms / 1e6, 1), "launches_per_block": launches,
            "kernels": [{1: "generic", 2: "tiled", 3: "pipe"}[layer.info["kernel"]] for layer in layers],
            "data": "synthetic weights at Table-1 densities (PAPER.md L364-370)"}
    print(json.dumps(line), flush=True)
    blk.close()


def run_resize(N, Hin, Win, reps):
    """Resize-Conv-Relu-Maxpool: the c3 layer (64 -> 64 ch, 56x56,
    90% sparse) fed by a bilinear resize of an Hin x Win input."""
    import torch
    from paper_2005_04091_b200 import SparseConv2d
    cfg = synthgen.CONFIGS["c3"].with_batch(N)
    Lr = synthgen.make_layer(cfg, with_input=False)
    c = Lr.csr
    layer = SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values,
                         synthgen.make_bias(cfg.F, 7300))
    xs = [torch.from_numpy(synthgen.make_input((N, cfg.C, Hin, Win), 7400 + k)).cuda() for k in range(3)]
    for i in range(3):
        layer.resize_fused_relu_maxpool(xs[i % 3], with_argmax=False)
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        layer.resize_fused_relu_maxpool(xs[i % 3], with_argmax=False)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    flops = cfg.useful_flops
    print(json.dumps({"block": "resize_conv_relu_maxpool", "N": N, "input_hw": [Hin, Win],
                      "conv_hw": [cfg.H, cfg.W], "density": cfg.density, "ms": round(ms, 4),
                      "images_per_s": round(N / ms * 1e3, 1), "useful_gflops": round(flops / ms / 1e6, 1),
                      "launches_per_block": 1 + int(layer.info["launches_per_call"])}), flush=True)
    layer.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    run("resnet20_block10", RESNET20_BLOCK10, 256, a.reps, "resnet")
    run("vgg16_block10", VGG16_BLOCK10, 16, a.reps, "vgg")
    run_resize(32, 112, 112, a.reps)


if __name__ == "__main__":
    main()
