#!/usr/bin/env python
"""Benchmark of the CSR sparse direct convolution hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl native|reference]

A step = one forward of the whole hot path over one batch (SURVEY.md §8(a)
a4-a6: staging, sparse accumulation, epilogue) with the plan (a1-a3: validate,
decode, group; a7: CSR broadcast) built once beforehand and reported as
``create_ms``.  Workload (N=1): config c2 of BASELINE.json — N=32 C=F=64 56x56
K=3 pad 1, 80% random sparsity, conv only — the configuration the north-star
gate is quoted on.  Under torchrun each rank runs its own c2 batch (weak
scaling, no collective in the timed region).

Timing: W untimed warm-up steps, then EXACTLY K steps bracketed by a barrier +
cuda synchronize, CUDA events on the launching stream, max over ranks.  The
inputs rotate over enough buffer sets that each step's 51 MB working set has
been evicted from the 126 MB L2 by the time it is reused.

--impl reference times the CPU oracle (oracle/, the reference arm of this
paper-only tier) on this host's cores on a bounded sample of the same
workload, in the same unit.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402

METRIC = "effective GFLOP/s (nnz FLOPs) & images/s per sparse conv layer, 1/2/4/8 B200, % roofline"
L2_BYTES = 126 * 1024 * 1024
SM_COUNT = 148
FP32_LANES_PER_SM = 128


def _measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def fp32_peak_tflops():
    """FP32 FFMA peak = 148 SM x 128 lanes x 2 FLOP x max SM clock."""
    mp = _measured_peaks()
    mhz = float(mp.get("sm_max_mhz", 1965.0))
    return SM_COUNT * FP32_LANES_PER_SM * 2 * mhz * 1e6 / 1e12, mhz, ("MEASURED_PEAKS.json sm_max_mhz"
                                                                   if "sm_max_mhz" in mp else "nominal 1965 MHz")


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML absent
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _cpu_oracle_sample(cfg, L, budget_s: float, nthreads: int):
    """Time the oracle (as it stands) on a bounded sample of whole images of ``cfg``:
    passes over (up to) the workload's N images until about ``budget_s`` of CPU work."""
    import oracle
    c = L.csr
    args = (cfg.F, cfg.K, cfg.stride, cfg.pad, c.rowptr, c.colidx, c.values, L.bias)
    fn = oracle.fused_f32 if cfg.fused else oracle.conv_f32
    t0 = time.perf_counter()
    fn(L.x[:1], *args, nthreads=nthreads)
    t1 = max(time.perf_counter() - t0, 1e-6)
    n_target = max(1, int(budget_s / t1))
    done, dt = 0, 0.0
    while done < n_target:
        n = min(cfg.N, n_target - done)
        t0 = time.perf_counter()
        fn(L.x[:n], *args, nthreads=nthreads)
        dt += time.perf_counter() - t0
        done += n
    flops = 2 * c.nnz * done * cfg.Ho * cfg.Wo
    return flops / dt / 1e9, done, dt


def run_reference(args, cfg):
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    L = synthgen.make_layer(cfg)
    nthreads = oracle.default_threads()
    # each step: a bounded sample of the workload's images, sized so that the whole
    # --steps K --warmup W run takes about two minutes of CPU time
    c = L.csr
    args_o = (cfg.F, cfg.K, cfg.stride, cfg.pad, c.rowptr, c.colidx, c.values, L.bias)
    t0 = time.perf_counter()
    oracle.conv_f32(L.x[:1], *args_o, nthreads=nthreads)
    t1 = time.perf_counter() - t0
    n_img = max(1, min(cfg.N, int(120.0 / ((args.steps + args.warmup) * max(t1, 1e-6)))))
    fn = oracle.fused_f32 if cfg.fused else oracle.conv_f32
    for _ in range(args.warmup):
        fn(L.x[:n_img], *args_o, nthreads=nthreads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn(L.x[:n_img], *args_o, nthreads=nthreads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    flops = 2 * c.nnz * n_img * cfg.Ho * cfg.Wo * args.steps
    value = flops / total / 1e9
    sample = f"{n_img} of {cfg.N} images of {cfg.name} per step, {nthreads} threads"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config(cfg, world, "CPU oracle; no GPU"),
        "images_per_s": round(n_img * args.steps / total, 3),
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": nthreads,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(cfg, world, l2note):
    return {"workload": f"{cfg.name}: {cfg.note}", "N_per_gpu": cfg.N, "C": cfg.C, "H": cfg.H,
            "W": cfg.W, "F": cfg.F, "K": cfg.K, "stride": cfg.stride, "pad": cfg.pad,
            "sparsity": round(1 - cfg.density, 4), "nnz": cfg.nnz, "fused": cfg.fused,
            "bias": cfg.bias, "global_batch": cfg.N * world,
            "parallelism": f"batch-sharded dp{world}", "l2": l2note}


def run_native(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2005_04091_b200 import SparseConv2d, spconv
    from paper_2005_04091_b200.parallel import broadcast_csr

    world, rank, local = _dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py native arm needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    # ---- plan (a1-a3, a7 broadcast): once, outside the timed region
    L = synthgen.make_layer(cfg, with_input=False)
    t0 = time.perf_counter()
    if world > 1:
        rp, ci, vv, b = broadcast_csr(L.csr.rowptr if rank == 0 else None,
                                      L.csr.colidx if rank == 0 else None,
                                      L.csr.values if rank == 0 else None,
                                      L.bias if rank == 0 else None, cfg.F, dev)
    else:
        rp, ci, vv, b = L.csr.rowptr, L.csr.colidx, L.csr.values, L.bias
    layer = SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, cfg.K, cfg.stride, cfg.pad, rp, ci, vv, b,
                         device=local, kernel=args.kernel, rows_per_group=args.rows)
    torch.cuda.synchronize()
    create_ms = 1e3 * (time.perf_counter() - t0)
    info = layer.info

    # ---- inputs: this rank's images (counter-based generator, offset by rank)
    shape = (cfg.N, cfg.C, cfg.H, cfg.W)
    x_host = np.empty(shape, np.float32)
    n_el = x_host.size
    u = synthgen.splitmix64(synthgen.seed_of(cfg.k, 2),
                            np.arange(rank * n_el, (rank + 1) * n_el, dtype=np.uint64))
    x_host[...] = synthgen.unit_float(u).reshape(shape)
    out_shape = layer.output_shape(cfg.N, cfg.fused)
    in_bytes = x_host.nbytes
    out_bytes = int(np.prod(out_shape)) * 4 * (2 if cfg.fused else 1)
    nsets = max(2, math.ceil(3 * L2_BYTES / (in_bytes + out_bytes)))
    xs = [torch.from_numpy(x_host).to(dev) for _ in range(nsets)]
    ys = [torch.empty(out_shape, dtype=torch.float32, device=dev) for _ in range(nsets)]
    ams = [torch.empty(out_shape, dtype=torch.int32, device=dev) for _ in range(nsets)] if cfg.fused else None
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def step(i):
        j = i % nsets
        if cfg.fused:
            spconv.spconv_fused_relu_maxpool(layer.plan, cfg.N, xs[j].data_ptr(), ys[j].data_ptr(),
                                             ams[j].data_ptr(), sh)
        else:
            spconv.spconv_forward(layer.plan, cfg.N, xs[j].data_ptr(), ys[j].data_ptr(), sh)

    for i in range(args.warmup):
        step(i)
    # (1) the timed region: K back-to-back steps bracketed by two events only (events
    # between launches would sit in the stream between kernels and add ~5 us a step,
    # and would stop a launch from overlapping its predecessor's tail)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_start.record(stream)
        for i in range(args.steps):
            step(args.warmup + i)
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    # (2) the kernel's launch duration for the roofline: the same steps again, each
    # launch bracketed by its own events on the launching stream
    nk = min(args.steps, 200)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nk)]
    torch.cuda.synchronize()
    for i in range(nk):
        ev[i][0].record(stream)
        step(args.warmup + args.steps + i)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    per_launch = [a.elapsed_time(b) for a, b in ev]
    kern_ms = sum(per_launch) / len(per_launch)
    if world > 1:
        t = torch.tensor([elapsed_ms, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, kern_ms = float(t[0]), float(t[1])
    ms_per_step = elapsed_ms / args.steps
    flops_per_step = cfg.useful_flops  # per rank
    value = flops_per_step * world / (ms_per_step * 1e-3) / 1e9
    images_per_s = cfg.N * world / (ms_per_step * 1e-3)

    # ---- end to end through the C-ABI with host buffers (H2D + forward + D2H per step)
    pin_x = torch.from_numpy(x_host).pin_memory().numpy()
    pin_y = torch.empty(out_shape, dtype=torch.float32).pin_memory().numpy()
    pin_a = torch.empty(out_shape, dtype=torch.int32).pin_memory().numpy() if cfg.fused else None
    e2e_steps = max(3, min(args.steps, 30))
    for _ in range(2):
        spconv.spconv_forward_host(layer.plan, cfg.N, pin_x, pin_y, cfg.fused, pin_a)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        spconv.spconv_forward_host(layer.plan, cfg.N, pin_x, pin_y, cfg.fused, pin_a)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    e2e_value = flops_per_step * world / e2e_s / 1e9

    # ---- optional: forward + all-gather of the outputs (the a7 collective), not the headline
    gather_ms = None
    if world > 1:
        from paper_2005_04091_b200.parallel import gather_output
        full = None
        for _ in range(3):
            step(0)
            full = gather_output(ys[0], cfg.N * world)
        torch.cuda.synchronize()
        dist.barrier()
        a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        reps = 10
        for _ in range(reps):
            step(0)
            full = gather_output(ys[0], cfg.N * world)
        bb.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(bb) / reps], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gather_ms = float(t[0])
        del full

    peak, mhz, peak_src = fp32_peak_tflops()
    achieved = flops_per_step / (kern_ms * 1e-3) / 1e12
    traffic = _profiled_traffic(cfg.name, info)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded SplitMix64, BASELINE.json c2 shape; random pruning)",
        "config": _config(cfg, world, f"rotating {nsets} input/output sets "
                                       f"({nsets * (in_bytes + out_bytes) / 2**20:.0f} MiB > 126 MiB L2)"),
        "images_per_s": round(images_per_s, 1),
        "kernel": {1: "generic", 2: "tiled", 3: "pipe"}[info["kernel"]],
        "rows_per_group": int(info["rows_per_group"]),
        "kernel_ms": round(kern_ms, 5),
        "create_ms": round(create_ms, 3),
        "roofline": {"bound": "alu", "achieved": round(achieved, 3), "peak": round(peak, 2),
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": f"148 SM x 128 FP32 lanes x 2 x {mhz:.0f} MHz ({peak_src})",
                     "algorithmic_flops_per_launch": flops_per_step,
                     "duration": "mean of per-launch CUDA event pairs on the launching stream "
                                 "(a separate pass: the events serialise the launches; the timed "
                                 "region lets each launch overlap its predecessor's tail via "
                                 "programmatic dependent launch)"},
        "e2e": {"value": round(e2e_value, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": in_bytes,
                "d2h_bytes_per_step": out_bytes, "steps": e2e_steps,
                "api": "spconv_forward_host (pinned host buffers)"},
        "clocks": clk.summary(),
        "gpu_launches": args.steps * int(info["launches_per_call"]),
    }
    if gather_ms is not None:
        line["forward_allgather_ms"] = round(gather_ms, 4)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Lx = synthgen.make_layer(cfg)
        import oracle
        nthreads = oracle.default_threads()
        v, n_img, dt = _cpu_oracle_sample(cfg, Lx, args.cpu_budget, nthreads)
        line["cpu_baseline"] = {"value": round(v, 3), "unit": "GFLOP/s", "cores": nthreads,
                                "kind": "oracle",
                                "sample": f"{n_img} images of {cfg.name} (passes over its N={cfg.N} "
                                          f"images), {dt:.1f} s, FP32-ordered oracle"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    layer.close()
    return 0


def _profiled_traffic(name, info):
    """dram read+write bytes per launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(name)
        if e and e.get("kernel") == {1: "generic", 2: "tiled", 3: "pipe"}[info["kernel"]]:
            return e.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="c2", choices=sorted(synthgen.CONFIGS))
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "pipe", "tiled", "generic"])
    ap.add_argument("--rows", type=int, default=0, help="rows per group R (0 = library default)")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle CPU work (estimate)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    cfg = synthgen.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_native(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
