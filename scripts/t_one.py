import sys, numpy as np, torch
sys.path.insert(0, '.')
import synthgen
from paper_2005_04091_b200 import SparseConv2d
cfg = synthgen.CONFIGS[sys.argv[1] if len(sys.argv)>1 else "c1"]
L = synthgen.make_layer(cfg.with_batch(1))
c = L.csr
layer = SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, cfg.K, cfg.stride, cfg.pad, c.rowptr, c.colidx, c.values, None, device=0, kernel="tiled")
y = layer(torch.from_numpy(L.x).cuda()); torch.cuda.synchronize(); print("ok", y.abs().sum().item())
