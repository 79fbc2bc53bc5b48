"""A/B: back-to-back c2 forwards with only start/end events (no per-launch events),
SPCONV_PDL=0 vs default (programmatic dependent launch)."""
import os, subprocess, sys
if len(sys.argv) == 1:
    for v in ("0", "1", "0", "1"):
        subprocess.run([sys.executable, __file__, "run"], env=dict(os.environ, SPCONV_PDL=v))
    sys.exit(0)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, synthgen
from paper_2005_04091_b200 import spconv
cfg = synthgen.CONFIGS["c2"]
L = synthgen.make_layer(cfg)
layer = spconv.SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, 3, 1, 1, L.csr.rowptr, L.csr.colidx, L.csr.values)
xs = [torch.from_numpy(L.x).cuda() for _ in range(8)]
ys = [torch.empty(layer.output_shape(cfg.N, False), device="cuda") for _ in range(8)]
sh = torch.cuda.current_stream().cuda_stream
def step(i): spconv.spconv_forward(layer.plan, cfg.N, xs[i % 8].data_ptr(), ys[i % 8].data_ptr(), sh)
for i in range(10): step(i)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); a.record()
for i in range(400): step(i)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 400
print(f"PDL={os.environ['SPCONV_PDL']}: {ms*1e3:.2f} us/step  {cfg.useful_flops/ms/1e9:.0f} GFLOP/s")
