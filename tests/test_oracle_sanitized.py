"""The host oracle under AddressSanitizer + UndefinedBehaviorSanitizer:
a subprocess with the ASan runtime preloaded runs every oracle entry point on small
seeded cases (conv f32/f64, fused, point queries, decode, CSR check incl. malformed
input, epilogue, resize, LSTM) and compares with the uninstrumented build bitwise.
Any out-of-bounds access or UB aborts the child (-fno-sanitize-recover)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import numpy as np, sys
sys.path.insert(0, ROOT)
import oracle, synthgen
assert oracle.SANITIZE
def run():
    out = []
    for name, N in (("c1", 2), ("c2", 1)):
        cfg = synthgen.CONFIGS[name].with_batch(N)
        if name == "c2":
            cfg = synthgen.LayerConfig(2, "c2s", 1, 6, 9, 11, 5, 3, 1, 1, 0.3, False, True)
        L = synthgen.make_layer(cfg)
        c = L.csr
        b = synthgen.make_bias(cfg.F, 5)
        args = (L.x, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values, b)
        y = oracle.conv_f32(*args); out.append(y)
        out.append(oracle.conv_f64(*args))
        p, a = oracle.fused_f32(*args); out += [p, a]
        pts = np.array([[0, 0, 0, 0], [N - 1, cfg.F - 1, y.shape[2] - 1, y.shape[3] - 1]], np.int64)
        out.append(oracle.conv_points_f32(*args, pts)); out.append(oracle.conv_points_f64(*args, pts))
        pts2 = np.array([[0, 0, 0, 0]], np.int64)
        v, ai = oracle.fused_points_f32(*args, pts2); out += [v, ai]
        out += list(oracle.decode(3, c.colidx))
        out.append(np.array([oracle.check_csr(cfg.F, cfg.C, 3, c.rowptr, c.colidx, c.values)]))
        bad = c.colidx.copy(); bad[0] = 10**6
        out.append(np.array([oracle.check_csr(cfg.F, cfg.C, 3, c.rowptr, bad, c.values)]))
        out.append(oracle.conv_ex_f32(*args, residual=y, relu=True))
    xr = synthgen.make_input((1, 2, 7, 9), 3)
    out.append(oracle.resize_bilinear_f32(xr, 5, 4))
    layers, xl = synthgen.make_lstm(2, 6, 4, 0.5, 3, 2)
    out.append(oracle.lstm_f64(xl, layers, 4))
    return out
res = run()
np.savez(OUT, *res)
'''


def test_oracle_under_asan_ubsan(tmp_path):
    asan = subprocess.run(["gcc", "-print-file-name=libasan.so"], capture_output=True, text=True).stdout.strip()
    ubsan = subprocess.run(["gcc", "-print-file-name=libubsan.so"], capture_output=True, text=True).stdout.strip()
    if not os.path.isabs(asan) or not os.path.exists(asan):
        pytest.skip("no libasan in this gcc")
    out_san, out_ref = tmp_path / "san.npz", tmp_path / "ref.npz"
    code = CHILD.replace("ROOT", repr(ROOT))
    env = dict(os.environ, ORACLE_SANITIZE="1", LD_PRELOAD=f"{asan}:{ubsan}",
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=1", UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    r = subprocess.run([sys.executable, "-c", code.replace("OUT", repr(str(out_san)))], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    assert "runtime error" not in r.stderr and "AddressSanitizer" not in r.stderr, r.stderr[-4000:]
    env2 = dict(os.environ)
    env2.pop("ORACLE_SANITIZE", None)
    code2 = code.replace("assert oracle.SANITIZE", "assert not oracle.SANITIZE")
    r2 = subprocess.run([sys.executable, "-c", code2.replace("OUT", repr(str(out_ref)))], env=env2,
                        capture_output=True, text=True, timeout=600)
    assert r2.returncode == 0, r2.stderr[-4000:]
    import numpy as np
    a, b = np.load(out_san), np.load(out_ref)
    assert a.files == b.files
    for k in a.files:
        assert np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)), k
