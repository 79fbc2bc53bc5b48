"""Run the randomised-shape parity cases one per subprocess (CUDA errors are sticky)
and print the first failing (case, kernel, shape)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
if len(sys.argv) == 1:
    for i in range(60):
        for kernel in ("auto", "pipe", "tiled"):
            r = subprocess.run([sys.executable, __file__, str(i), kernel], capture_output=True, text=True,
                               env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"))
            last = (r.stdout + r.stderr).strip().splitlines()[-1:] or [""]
            if r.returncode != 0:
                print("FAIL", i, kernel, last[0][:300])
    sys.exit(0)
import torch, synthgen, oracle
from paper_2005_04091_b200 import SparseConv2d
from paper_2005_04091_b200.spconv import SpconvError
rng = np.random.default_rng(20050409)
ci, kernel = int(sys.argv[1]), sys.argv[2]
for i in range(ci + 1):
    N = int(rng.integers(1, 6)); C = int(rng.integers(1, 40)); H = int(rng.integers(1, 40))
    W = int(rng.choice([int(rng.integers(1, 40)), 4 * int(rng.integers(1, 31))]))
    F = int(rng.integers(1, 70)); d = float(rng.choice([0.05, 0.2, 0.5, 1.0]))
seed = 9000 + 10 * ci
csr = synthgen.make_csr(F, C, 3, d, seed, seed + 1)
xh = synthgen.make_input((N, C, H, W), seed + 2)
b = synthgen.make_bias(F, seed + 3) if ci % 2 else None
print("case", ci, kernel, dict(N=N, C=C, H=H, W=W, F=F, d=d, bias=b is not None))
try:
    layer = SparseConv2d(C, H, W, F, 3, 1, 1, csr.rowptr, csr.colidx, csr.values, b, kernel=kernel)
except SpconvError as e:
    print("unsupported", e.status); sys.exit(0)
x = torch.from_numpy(xh).cuda()
y = layer(x).cpu().numpy()
ref = oracle.conv_f32(xh, F, 3, 1, 1, csr.rowptr, csr.colidx, csr.values, b)
assert np.array_equal(y.view(np.uint32), ref.view(np.uint32)), "conv mismatch"
if H >= 2 and W >= 2:
    p, am = layer.fused_relu_maxpool(x)
    rp, ra = oracle.fused_f32(xh, F, 3, 1, 1, csr.rowptr, csr.colidx, csr.values, b)
    assert np.array_equal(p.cpu().numpy().view(np.uint32), rp.view(np.uint32)), "fused mismatch"
    assert np.array_equal(am.cpu().numpy(), ra), "argmax mismatch"
print("ok")
