#!/usr/bin/env python
"""Benchmark of the CSR sparse direct convolution hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--scaling weak|strong]
                    [--impl native|reference]

A step = one forward of the whole hot path over one batch (SURVEY.md §8(a)
a4-a6: staging, sparse accumulation, epilogue) with the plan (a1-a3: validate,
decode, group; a7: CSR broadcast) built once beforehand and reported as
``create_ms`` / ``broadcast_ms``.  Workload (N=1): config c2 of BASELINE.json —
N=32 C=F=64 56x56 K=3 pad 1, 80% random sparsity, conv only — the
configuration the north-star gate is quoted on.

Multi-GPU: ``--gpus N`` with N > 1 and no WORLD_SIZE in the environment spawns N
ranks itself (torch.distributed.run, one process per GPU, NCCL); under torchrun
the world size must equal --gpus.  ``--scaling weak`` (default): every rank runs
its own full batch; ``--scaling strong``: the config's global batch is sharded
(contiguous images), e.g. c5's 256 images over 2/4/8 GPUs.  No
collective in the timed region; forward + all-gather and broadcast + create are
reported beside it.

Timing ("repeated 30 times and the median is reported"): W
untimed warm-ups, then EXACTLY K steps (default 100; the paper's 30 or more is the
intent, fewer are accepted and the median is over what was asked) between a barrier + cuda
synchronize on both sides; before every step the L2 is flushed (a write of 2x
the 126 MB L2, untimed) and the step itself is bracketed by CUDA events on the
launching stream; ``ms_per_step`` = the median step (max over ranks).  Also
reported: the warm-L2 median (same input re-used, no flush) and the steady-state
throughput of back-to-back launches on rotating inputs larger than the L2.

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


def host_cpu_info():
    """CPU model, logical and physical core counts of this host."""
    info = {"logical_cpus": os.cpu_count(), "affinity_cpus": len(os.sched_getaffinity(0))}
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        info["model"] = kv.get("Model name")
        cps = int(kv.get("Core(s) per socket", "0") or 0)
        sockets = int(kv.get("Socket(s)", "0") or 0)
        if cps and sockets:
            info["physical_cores"] = cps * sockets
    except Exception:  # pragma: no cover - lscpu absent
        pass
    return info


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


def run_reference(args, cfg, world=None):
    w, rank, _ = _dist_env()
    world = w if world is None else world
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
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config(cfg, world, "CPU oracle; no GPU", scaling=args.scaling),
        "images_per_s": round(n_img * args.steps / total, 3),
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": nthreads,
                         "kind": "oracle", "sample": sample, "host": host_cpu_info()},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config(cfg, world, l2note, n_local=None, global_batch=None, scaling="weak"):
    return {"workload": f"{cfg.name}: {cfg.note}", "N_per_gpu": cfg.N if n_local is None else n_local,
            "C": cfg.C, "H": cfg.H, "W": cfg.W, "F": cfg.F, "K": cfg.K, "stride": cfg.stride, "pad": cfg.pad,
            "sparsity": round(1 - cfg.density, 4), "nnz": cfg.nnz, "fused": cfg.fused,
            "bias": cfg.bias, "global_batch": cfg.N * world if global_batch is None else global_batch,
            "parallelism": f"batch-sharded dp{world} ({scaling} scaling)", "l2": l2note}


def rank_images(n_config: int, world: int, rank: int, scaling: str):
    """[b0, b1) global image indices of this rank and the global batch: weak scaling gives
    every rank the config's whole batch (images rank*N .. rank*N+N-1 of the counter
    stream); strong scaling splits the config's batch in contiguous shards."""
    from paper_2005_04091_b200.parallel import shard_bounds
    if scaling == "strong":
        b0, b1 = shard_bounds(n_config, world, rank)
        return b0, b1, n_config
    return rank * n_config, (rank + 1) * n_config, n_config * world


def _median_max(vals_ms, dev, world):
    """Median of this rank's per-step times, then the max over ranks."""
    import torch
    import torch.distributed as dist
    m = float(statistics.median(vals_ms))
    if world > 1:
        t = torch.tensor([m], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        m = float(t[0])
    return m


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
        if rank == 0:  # communicator init lines (NCCL version, ranks, transports) on rank 0
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()

    # ---- this rank's images: weak = the config's full batch per rank, strong = a
    # contiguous shard of the config's batch
    b0, b1, global_batch = rank_images(cfg.N, world, rank, args.scaling)
    n_local = b1 - b0
    lcfg = cfg.with_batch(max(n_local, 1))

    # ---- plan (a1-a3, a7 broadcast): once, outside the timed region
    L = synthgen.make_layer(cfg, with_input=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if world > 1:
        rp, ci, vv, b = broadcast_csr(L.csr.rowptr if rank == 0 else None,
                                      L.csr.colidx if rank == 0 else None,
                                      L.csr.values if rank == 0 else None,
                                      L.bias if rank == 0 else None, cfg.F, dev)
        torch.cuda.synchronize()
    else:
        rp, ci, vv, b = L.csr.rowptr, L.csr.colidx, L.csr.values, L.bias
    t1 = time.perf_counter()
    layer = SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, cfg.K, cfg.stride, cfg.pad, rp, ci, vv, b,
                         device=local, kernel=args.kernel, rows_per_group=args.rows)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    broadcast_ms, create_ms = 1e3 * (t1 - t0), 1e3 * (t2 - t1)
    info = layer.info

    # ---- inputs: the counter-based generator at this rank's global image indices
    shape = (n_local, cfg.C, cfg.H, cfg.W)
    x_host = np.empty(shape, np.float32)
    per_img = cfg.C * cfg.H * cfg.W
    u = synthgen.splitmix64(synthgen.seed_of(cfg.k, 2),
                            np.arange(b0 * per_img, b1 * per_img, dtype=np.uint64))
    x_host[...] = synthgen.unit_float(u).reshape(shape)
    out_shape = layer.output_shape(n_local, cfg.fused)
    in_bytes = x_host.nbytes
    out_bytes = int(np.prod(out_shape)) * 4 * (2 if cfg.fused else 1)
    nsets = max(2, math.ceil(3 * L2_BYTES / max(1, in_bytes + out_bytes)))
    xs = [torch.from_numpy(x_host).to(dev) for _ in range(nsets)]
    ys = [torch.empty(out_shape, dtype=torch.float32, device=dev) for _ in range(nsets)]
    ams = [torch.empty(out_shape, dtype=torch.int32, device=dev) for _ in range(nsets)] if cfg.fused else None
    flush_buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    launch = spconv.spconv_launch_info(layer.plan, n_local, cfg.fused, xs[0].data_ptr()) if n_local else {}

    def step(i):
        if n_local == 0:
            return
        j = i % nsets
        if cfg.fused:
            spconv.spconv_fused_relu_maxpool(layer.plan, n_local, xs[j].data_ptr(), ys[j].data_ptr(),
                                             ams[j].data_ptr(), sh)
        else:
            spconv.spconv_forward(layer.plan, n_local, xs[j].data_ptr(), ys[j].data_ptr(), sh)

    for i in range(args.warmup):
        step(i)
    # (1) the timed region (PAPER.md L436 protocol): K steps, each after an L2 flush and
    # between its own pair of events on the launching stream; median step, max over ranks
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    t_all0, t_all1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_all0.record(stream)
        for i in range(args.steps):
            flush_buf.zero_()
            ev[i][0].record(stream)
            step(args.warmup + i)
            ev[i][1].record(stream)
        t_all1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_step = [a.elapsed_time(bb) for a, bb in ev]
    ms_per_step = _median_max(per_step, dev, world)
    region_ms = t_all0.elapsed_time(t_all1)

    # (2) warm-L2 median: the same input again and again, no flush (30 reps)
    wev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
    torch.cuda.synchronize()
    for a, bb in wev:
        a.record(stream)
        step(0)
        bb.record(stream)
    torch.cuda.synchronize()
    warm_ms = _median_max([a.elapsed_time(bb) for a, bb in wev], dev, world)

    # (3) steady state: back-to-back launches on rotating inputs larger than the L2, two
    # events only (consecutive launches overlap via programmatic dependent launch)
    nb = max(30, min(args.steps, 300))
    a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a.record(stream)
    for i in range(nb):
        step(i)
    bb.record(stream)
    torch.cuda.synchronize()
    steady_ms = _median_max([a.elapsed_time(bb) / nb], dev, world)

    local_flops = 2 * cfg.nnz * n_local * cfg.Ho * cfg.Wo
    global_flops = 2 * cfg.nnz * global_batch * cfg.Ho * cfg.Wo
    value = global_flops / (ms_per_step * 1e-3) / 1e9
    images_per_s = global_batch / (ms_per_step * 1e-3)

    # ---- end to end through the C-ABI with host buffers (H2D + forward + D2H per step)
    e2e_steps = max(3, min(args.steps, 30))
    e2e_value, e2e_s = None, None
    if n_local:
        pin_x = torch.from_numpy(x_host).pin_memory().numpy()
        pin_y = torch.empty(out_shape, dtype=torch.float32).pin_memory().numpy()
        pin_a = torch.empty(out_shape, dtype=torch.int32).pin_memory().numpy() if cfg.fused else None
        for _ in range(2):
            spconv.spconv_forward_host(layer.plan, n_local, pin_x, pin_y, cfg.fused, pin_a)
    if world > 1:
        dist.barrier()
    tt0 = time.perf_counter()
    for _ in range(e2e_steps if n_local else 0):
        spconv.spconv_forward_host(layer.plan, n_local, pin_x, pin_y, cfg.fused, pin_a)
    e2e_s = (time.perf_counter() - tt0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    e2e_value = global_flops / e2e_s / 1e9

    # ---- forward + all-gather of the outputs (the a7 collective), beside the headline
    gather_ms = None
    if world > 1 and args.scaling == "strong":
        from paper_2005_04091_b200.parallel import gather_output
        for _ in range(3):
            step(0)
            full = gather_output(ys[0], cfg.N)
        torch.cuda.synchronize()
        dist.barrier()
        ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ga.record(stream)
        reps = 10
        for _ in range(reps):
            step(0)
            full = gather_output(ys[0], cfg.N)
        gb.record(stream)
        torch.cuda.synchronize()
        gather_ms = _median_max([ga.elapsed_time(gb) / reps], dev, world)
        del full

    peak, mhz, peak_src = fp32_peak_tflops()
    achieved = local_flops / (ms_per_step * 1e-3) / 1e12
    traffic = _profiled_traffic(cfg.name, info)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic (seeded SplitMix64, BASELINE.json {cfg.name} shape; random pruning)",
        "config": _config(cfg, world, f"L2 flushed before every timed step (write of {2 * L2_BYTES >> 20} MiB, "
                                      f"untimed); steady-state pass rotates {nsets} input/output sets "
                                      f"({nsets * (in_bytes + out_bytes) / 2**20:.0f} MiB)",
                          n_local=n_local, global_batch=global_batch, scaling=args.scaling),
        "images_per_s": round(images_per_s, 1),
        "timing": {"protocol": f"median of the K = {args.steps} per-step CUDA-event times, L2 flushed before "
                               "each (PAPER.md L436: median of 30 reps)",
                   "median_ms": round(ms_per_step, 5), "warm_l2_median_ms": round(warm_ms, 5),
                   "steady_state_ms": round(steady_ms, 5),
                   "steady_state_value": round(global_flops / (steady_ms * 1e-3) / 1e9, 2),
                   "timed_region_ms": round(region_ms, 3)},
        "kernel": {1: "generic", 2: "tiled", 3: "pipe", 4: "dense"}[info["kernel"]],
        "rows_per_group": int(info["rows_per_group"]),
        "launch": launch,
        "kernel_ms": round(ms_per_step, 5),
        "create_ms": round(create_ms, 3),
        "broadcast_ms": round(broadcast_ms, 3),
        "roofline": {"bound": "alu", "achieved": round(achieved, 3), "peak": round(peak, 2),
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": f"148 SM x 128 FP32 lanes x 2 x {mhz:.0f} MHz ({peak_src}); "
                                    "FFMA/FFMA2 probe: profiles/r02_ffma_peak_probe.log",
                     "algorithmic_flops_per_launch": local_flops,
                     "duration": "median per-launch CUDA event time on the launching stream (the timed "
                                 "steps; one launch per step)"},
        "e2e": {"value": round(e2e_value, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": in_bytes,
                "d2h_bytes_per_step": out_bytes, "steps": e2e_steps,
                "api": "spconv_forward_host (pinned host buffers)"},
        "clocks": clk.summary(),
        "gpu_launches": args.steps * int(launch.get("launches", 1) if launch else 0),
    }
    if gather_ms is not None:
        line["forward_allgather_ms"] = round(gather_ms, 4)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Lx = synthgen.make_layer(cfg)
        import oracle
        nthreads = oracle.default_threads()
        v, n_img, dt = _cpu_oracle_sample(cfg, Lx, args.cpu_budget, nthreads)
        line["cpu_baseline"] = {"value": round(v, 3), "unit": "GFLOP/s", "cores": nthreads,
                                "kind": "oracle", "host": host_cpu_info(),
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
        if e and e.get("kernel") == {1: "generic", 2: "tiled", 3: "pipe", 4: "dense"}[info["kernel"]]:
            return e.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass
    return None


def _spawn(args_list, n):
    """Re-launch this script as n ranks (one process per GPU) under torch.distributed.run."""
    import socket
    import subprocess
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *args_list]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2", choices=sorted(synthgen.CONFIGS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "pipe", "tiled", "generic", "dense"])
    ap.add_argument("--rows", type=int, default=0, help="rows per group R (0 = library default)")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle CPU work (estimate)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.steps < 1:
        ap.error("--steps must be >= 1")
    cfg = synthgen.CONFIGS[args.config]
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus:
            ap.error(f"--gpus {args.gpus} disagrees with WORLD_SIZE={os.environ['WORLD_SIZE']}")
    elif args.gpus > 1:
        if args.impl == "reference":  # the CPU oracle arm: one process (rank 0's work)
            return run_reference(args, cfg, world=args.gpus)
        return _spawn(sys.argv[1:], args.gpus)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_native(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
