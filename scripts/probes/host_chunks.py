"""A/B: spconv_forward_host step time vs the number of pipelined chunks (c2, pinned)."""
import os, subprocess, sys, time
if len(sys.argv) == 1:
    for k in (1, 2, 3, 4, 6, 8, 12, 16):
        env = dict(os.environ, SPCONV_HOST_CHUNKS=str(k))
        subprocess.run([sys.executable, __file__, "run"], env=env)
    sys.exit(0)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synthgen
from paper_2005_04091_b200 import spconv
cfg = synthgen.CONFIGS[os.environ.get("CFG", "c2")]
L = synthgen.make_layer(cfg)
layer = spconv.SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, 3, 1, 1, L.csr.rowptr, L.csr.colidx, L.csr.values)
x = torch.from_numpy(L.x).pin_memory().numpy()
y = torch.empty(layer.output_shape(cfg.N, False), dtype=torch.float32).pin_memory().numpy()
for _ in range(3): spconv.spconv_forward_host(layer.plan, cfg.N, x, y, 0, None)
t0 = time.perf_counter()
for _ in range(30): spconv.spconv_forward_host(layer.plan, cfg.N, x, y, 0, None)
dt = (time.perf_counter() - t0) / 30
print(f"chunks={os.environ['SPCONV_HOST_CHUNKS']}: {dt*1e3:.3f} ms/step  {cfg.useful_flops/dt/1e9:.0f} GFLOP/s e2e")
