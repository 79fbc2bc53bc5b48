import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synthgen
from paper_2005_04091_b200.lstm import WAVEFRONT, SparseLSTM
L, D, H, T, B, d = [float(v) if '.' in v else int(v) for v in sys.argv[1:7]]
layers, x = synthgen.make_lstm(L, D, H, d, T, B)
net = SparseLSTM(D, H, layers)
h = net(torch.from_numpy(x).cuda(), WAVEFRONT)
torch.cuda.synchronize(); print("ok", float(h.abs().sum()))
