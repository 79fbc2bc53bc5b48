"""Host time per C-ABI call (no synchronisation inside the loop) for a tiny layer, per
library build (SPCONV_LIB): the launch-path overhead a back-to-back caller pays."""
import json, os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch, synthgen
    from paper_2005_04091_b200 import spconv
    name, kernel = sys.argv[2], sys.argv[3]
    cfg = synthgen.CONFIGS[name]
    L = synthgen.make_layer(cfg)
    layer = spconv.SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, 3, 1, 1, L.csr.rowptr, L.csr.colidx, L.csr.values,
                                kernel=kernel)
    x = torch.from_numpy(L.x).cuda()
    y = torch.empty(layer.output_shape(cfg.N), device="cuda")
    sh = torch.cuda.current_stream().cuda_stream
    for _ in range(50):
        spconv.spconv_forward(layer.plan, cfg.N, x.data_ptr(), y.data_ptr(), sh)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        spconv.spconv_forward(layer.plan, cfg.N, x.data_ptr(), y.data_ptr(), sh)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"lib": os.environ.get("SPCONV_LIB", "default").split("/")[-1], "config": name, "kernel": kernel,
                      "host_us_per_call": round((t1 - t0) / n * 1e6, 2), "wall_us_per_call": round((t2 - t0) / n * 1e6, 2)}), flush=True)
    sys.exit(0)
for lib in sys.argv[1].split(","):
    for name, kernel in (("c1", "pipe"), ("c1", "auto"), ("c2", "pipe"), ("c4_95", "pipe")):
        subprocess.run([sys.executable, __file__, "child", name, kernel], env=dict(os.environ, SPCONV_LIB=os.path.abspath(lib)),
                       timeout=300)
