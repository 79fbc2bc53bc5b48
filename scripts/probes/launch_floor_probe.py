"""Floor of the bench protocol for a tiny launch: the flushed / warm per-step event time
of a trivial kernel (a 4-byte fill) measured exactly as bench.py times one step
(L2 flush by a 252 MiB write, then start event, launch, end event; median of 100)."""
import json
import statistics
import torch

flush = torch.empty(252 * 2**20 // 4, dtype=torch.float32, device="cuda")
t = torch.empty(1, device="cuda")
for mode in ("flushed", "warm"):
    ts = []
    for i in range(110):
        if mode == "flushed":
            flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t.fill_(1.0)
        b.record()
        b.synchronize()
        if i >= 10:
            ts.append(a.elapsed_time(b) * 1000)
    print(json.dumps({"mode": mode, "median_us": round(statistics.median(ts), 2), "min_us": round(min(ts), 2)}))
