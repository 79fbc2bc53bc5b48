"""A/B of the end-to-end host-buffer entry point (spconv_forward_host) across library
builds (SPCONV_LIB) and chunk counts: pinned host buffers, median of 15 calls."""
import json, os, statistics, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np, torch, synthgen
    from paper_2005_04091_b200 import spconv
    cfg = synthgen.CONFIGS[sys.argv[2]]
    L = synthgen.make_layer(cfg)
    layer = spconv.SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, 3, 1, 1, L.csr.rowptr, L.csr.colidx, L.csr.values, L.bias)
    oshape = layer.output_shape(cfg.N, cfg.fused)
    px = torch.from_numpy(L.x).pin_memory().numpy()
    py = torch.empty(oshape, dtype=torch.float32).pin_memory().numpy()
    pa = torch.empty(oshape, dtype=torch.int32).pin_memory().numpy() if cfg.fused else None
    for _ in range(3):
        spconv.spconv_forward_host(layer.plan, cfg.N, px, py, cfg.fused, pa)
    ts = []
    for _ in range(15):
        t0 = time.perf_counter()
        spconv.spconv_forward_host(layer.plan, cfg.N, px, py, cfg.fused, pa)
        ts.append(time.perf_counter() - t0)
    ms = statistics.median(ts) * 1e3
    print(json.dumps({"lib": os.environ.get("SPCONV_LIB", "default"), "chunks": os.environ.get("SPCONV_HOST_CHUNKS"),
                      "config": cfg.name, "ms": round(ms, 4), "tflops": round(cfg.useful_flops / ms / 1e9, 3),
                      "in_MB": px.nbytes / 1e6}), flush=True)
    sys.exit(0)
libs = sys.argv[1].split(",") if len(sys.argv) > 1 and sys.argv[1] else [""]
configs = os.environ.get("E2E_CONFIGS", "c2,c4_80").split(",")
chunk_counts = os.environ.get("E2E_CHUNKS", ",1,4,8,16").split(",")
for cfg in configs:
    for lib in libs:
        for ch in chunk_counts:
            env = dict(os.environ)
            if lib:
                env["SPCONV_LIB"] = os.path.abspath(lib)
            if ch:
                env["SPCONV_HOST_CHUNKS"] = ch
            subprocess.run([sys.executable, __file__, "child", cfg], env=env, timeout=600)
