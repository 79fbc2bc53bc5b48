#!/usr/bin/env python
"""Small end-to-end invocations for compute-sanitizer:
conv + fused + epilogue + resize on c1/c2-shaped layers through every kernel and
staging path, and a small LSTM.  Exit code 0 if every output matches the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synthgen  # noqa: E402
from paper_2005_04091_b200 import SparseConv2d  # noqa: E402


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def check(cfg, kernel):
    L = synthgen.make_layer(cfg)
    c = L.csr
    b = synthgen.make_bias(cfg.F, 77)
    layer = SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values, b, kernel=kernel)
    x = torch.from_numpy(L.x).cuda()
    args = (L.x, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values, b)
    ok = np.array_equal(bits(layer(x).cpu().numpy()), bits(oracle.conv_f32(*args)))
    p, am = layer.fused_relu_maxpool(x)
    rp, ra = oracle.fused_f32(*args)
    ok &= np.array_equal(bits(p.cpu().numpy()), bits(rp)) and np.array_equal(am.cpu().numpy(), ra)
    r = torch.from_numpy(synthgen.make_input(tuple(layer.output_shape(cfg.N)), 78)).cuda()
    y = layer.forward_ex(x, relu=True, residual=r).cpu().numpy()
    ok &= np.array_equal(bits(y), bits(oracle.conv_ex_f32(*args, residual=r.cpu().numpy(), relu=True)))
    layer.close()
    return ok


def main():
    good = True
    for name, N in (("c1", 1), ("c2", 2), ("c4_80", 2)):
        for kernel in ("pipe", "tiled", "generic"):
            ok = check(synthgen.CONFIGS[name].with_batch(N), kernel)
            print(name, kernel, "ok" if ok else "MISMATCH", flush=True)
            good &= ok
    os.environ["SPCONV_PIPE_STAGING"] = "cp"
    ok = check(synthgen.CONFIGS["c2"].with_batch(1), "pipe")
    print("c2 pipe cp.async", "ok" if ok else "MISMATCH")
    good &= ok
    del os.environ["SPCONV_PIPE_STAGING"]
    # ordered stream-K at R = 4 (c2 N=23: 162 units on 148 CTAs, arrival tickets,
    # park / resume, walks split inside a stage)
    ok = check(synthgen.CONFIGS["c2"].with_batch(23), "pipe")
    print("c2 23 pipe R=4 stream-K", "ok" if ok else "MISMATCH", flush=True)
    good &= ok
    # R = 2 rows per group (11-12 warps per CTA), incl. ordered stream-K (c2 N=23)
    os.environ["SPCONV_PIPE_R"] = "2"
    for name, N in (("c2", 2), ("c2", 23), ("c4_50", 2)):
        ok = check(synthgen.CONFIGS[name].with_batch(N), "pipe")
        print(name, N, "pipe R=2", "ok" if ok else "MISMATCH", flush=True)
        good &= ok
    del os.environ["SPCONV_PIPE_R"]
    from paper_2005_04091_b200.lstm import SEQUENTIAL, WAVEFRONT, SparseLSTM
    layers, xl = synthgen.make_lstm(2, 24, 16, 0.3, 4, 3)
    net = SparseLSTM(24, 16, layers)
    hw = net(torch.from_numpy(xl).cuda(), WAVEFRONT).cpu().numpy()
    hs = net(torch.from_numpy(xl).cuda(), SEQUENTIAL).cpu().numpy()
    ok = np.array_equal(bits(hw), bits(hs)) and np.abs(hw - oracle.lstm_f64(xl, layers, 16)).max() < 1e-5
    print("lstm", "ok" if ok else "MISMATCH")
    good &= ok
    net.close()
    # batch >= 32: the z-staged kernel (cp.async ring, entries staged per chunk)
    layers, xl = synthgen.make_lstm(2, 100, 48, 0.2, 3, 36)
    net = SparseLSTM(100, 48, layers)
    hw = net(torch.from_numpy(xl).cuda(), WAVEFRONT).cpu().numpy()
    hs = net(torch.from_numpy(xl).cuda(), SEQUENTIAL).cpu().numpy()
    ok = np.array_equal(bits(hw), bits(hs)) and np.abs(hw - oracle.lstm_f64(xl, layers, 48)).max() < 1e-5
    print("lstm staged", "ok" if ok else "MISMATCH")
    good &= ok
    net.close()
    torch.cuda.synchronize()
    sys.exit(0 if good else 1)


if __name__ == "__main__":
    main()
