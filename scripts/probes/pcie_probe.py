"""Probe: pinned H2D / D2H bandwidth alone and concurrently (PCIe duplex) on the box."""
import torch, time
n = 25690112 // 4
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, device="cuda"); d_out = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def h2d():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
def both(): h2d(); d2h()
def chunks(k):
    def f():
        m = n // k
        for i in range(k):
            with torch.cuda.stream(s1): d_in[i*m:(i+1)*m].copy_(h_in[i*m:(i+1)*m], non_blocking=True)
            with torch.cuda.stream(s2): h_out[i*m:(i+1)*m].copy_(d_out[i*m:(i+1)*m], non_blocking=True)
    return f
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both), ("both_chunk8", chunks(8))):
    dt = t(fn)
    print(f"{name}: {dt*1e3:.3f} ms  ({n*4/dt/1e9:.1f} GB/s per direction)")
