"""Pins for the CPU oracle (no GPU).  Each test checks oracle/ against something
other than itself: hand-worked values, a separately written brute-force dense
convolution, torch's float64 conv2d / max_pool2d library routines, exact
integer arithmetic, closed forms and invariants."""
import numpy as np
import pytest
import torch

import oracle
import synthgen
from tests._util import (allclose_contract, bits, brute_dense_f32, csr_from_dense, densify,
                         load_golden)

GOLD = load_golden("hand_examples.json")


def _ex(name):
    return next(e for e in GOLD["examples"] if e["name"] == name)


def _x(e):
    return np.array(e["x"], np.float32).reshape(e["N"], e["C"], e["H"], e["W"])


# ---------------------------------------------------------------- hand examples
@pytest.mark.parametrize("name", ["A", "B", "C", "D"])
def test_hand_examples_conv(name):
    e = _ex(name)
    y = oracle.conv_f32(_x(e), e["F"], e["K"], e["stride"], e["pad"], e["rowptr"], e["colidx"],
                        e["values"])
    want = np.array(e["conv"], np.float32).reshape(y.shape)
    assert np.array_equal(y, want), (y, want)
    y64 = oracle.conv_f64(_x(e), e["F"], e["K"], e["stride"], e["pad"], e["rowptr"], e["colidx"],
                          e["values"])
    assert np.array_equal(y64, want.astype(np.float64))


@pytest.mark.parametrize("name", ["A", "B"])
def test_hand_examples_fused(name):
    e = _ex(name)
    args = (_x(e), e["F"], e["K"], e["stride"], e["pad"], e["rowptr"], e["colidx"], e["values"])
    p, am = oracle.fused_f32(*args, bias=np.array([e["fused_bias"]], np.float32))
    assert np.array_equal(p[0, 0], np.array(e["fused_pool"], np.float32))
    assert np.array_equal(am[0, 0], np.array(e["fused_argmax"], np.int32))
    p, am = oracle.fused_f32(*args)
    assert np.array_equal(p[0, 0], np.array(e["fused_nobias_pool"], np.float32))
    assert np.array_equal(am[0, 0], np.array(e["fused_nobias_argmax"], np.int32))


@pytest.mark.parametrize("win", GOLD["pool_windows"], ids=lambda w: w["name"])
def test_pool_window_rules(win):
    # 1x1 identity filter, pad 0: conv == input, so the 2x2 window is pooled as given.
    x = np.array(win["window"], np.float32).reshape(1, 1, 2, 2)
    p, am = oracle.fused_f32(x, 1, 1, 1, 0, [0, 1], [0], [1.0])
    assert p.item() == win["max"] and am.item() == win["argmax"]


# ---------------------------------------------------------------- decode
@pytest.mark.parametrize("C,K", [(1, 1), (3, 3), (17, 5), (256, 3), (64, 7)])
def test_decode_matches_numpy_flattening(C, K):
    # numpy's reshape of (C, K, K) -> (C*K*K) is the flattening of PAPER.md L391.
    cols = np.arange(C * K * K, dtype=np.int32)
    c, ky, kx = oracle.decode(K, cols)
    cc, yy, xx = np.unravel_index(cols, (C, K, K))
    assert np.array_equal(c, cc) and np.array_equal(ky, yy) and np.array_equal(kx, xx)


# ---------------------------------------------------------------- brute force dense
CASES = [
    # N, C, H, W, F, K, stride, pad, density
    (1, 1, 5, 5, 1, 3, 1, 1, 1.0),
    (2, 3, 7, 6, 4, 3, 1, 1, 0.2),
    (1, 4, 9, 9, 5, 3, 2, 1, 0.5),
    (2, 2, 8, 5, 3, 5, 1, 2, 0.3),
    (1, 5, 6, 6, 6, 1, 1, 0, 0.6),
    (1, 3, 10, 7, 2, 7, 2, 3, 0.1),
    (3, 2, 4, 4, 3, 3, 1, 0, 0.9),
    (1, 8, 12, 12, 8, 3, 1, 1, 0.0),   # nnz = 0
    (2, 6, 11, 13, 7, 3, 1, 2, 0.05),  # pad 2 -> larger output
]


def _rand_layer(case, seed, integer=False, bias=True):
    N, C, H, W, F, K, s, p, d = case
    csr = synthgen.make_csr(F, C, K, d, seed, seed + 1, integer=integer)
    x = synthgen.make_input((N, C, H, W), seed + 2, integer=integer)
    b = synthgen.make_bias(F, seed + 3, integer=integer) if bias else None
    return csr, x, b


@pytest.mark.parametrize("case", CASES)
def test_oracle_equals_brute_dense_bitwise(case):
    N, C, H, W, F, K, s, p, d = case
    csr, x, b = _rand_layer(case, 1000 + CASES.index(case) * 17)
    y = oracle.conv_f32(x, F, K, s, p, csr.rowptr, csr.colidx, csr.values, b)
    wd = densify(F, C, K, csr.rowptr, csr.colidx, csr.values)
    yb = brute_dense_f32(x, wd, b, s, p)
    assert y.shape == yb.shape
    assert np.array_equal(bits(y), bits(yb))


def test_zero_sparsity_equals_dense_conv():
    # 0% sparsity: a fully dense random filter bank, CSR from dense -> same as brute dense.
    rng = np.random.default_rng(7)
    w = rng.uniform(-1, 1, (4, 3, 3, 3)).astype(np.float32)
    w[w == 0] = 0.5
    x = rng.uniform(-1, 1, (2, 3, 9, 8)).astype(np.float32)
    rp, ci, vv = csr_from_dense(w)
    assert rp[-1] == w.size
    y = oracle.conv_f32(x, 4, 3, 1, 1, rp, ci, vv)
    assert np.array_equal(bits(y), bits(brute_dense_f32(x, w, None, 1, 1)))


@pytest.mark.parametrize("case", CASES)
def test_oracle_f64_vs_torch_conv2d(case):
    N, C, H, W, F, K, s, p, d = case
    csr, x, b = _rand_layer(case, 2000 + CASES.index(case) * 13)
    y = oracle.conv_f64(x, F, K, s, p, csr.rowptr, csr.colidx, csr.values, b)
    wd = densify(F, C, K, csr.rowptr, csr.colidx, csr.values)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(wd).double(),
                                     torch.from_numpy(b).double(), stride=s, padding=p).numpy()
    assert y.shape == ref.shape
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("case", CASES)
def test_integer_mode_exact_vs_torch(case):
    N, C, H, W, F, K, s, p, d = case
    csr, x, b = _rand_layer(case, 3000 + CASES.index(case), integer=True)
    y = oracle.conv_f32(x, F, K, s, p, csr.rowptr, csr.colidx, csr.values, b)
    wd = densify(F, C, K, csr.rowptr, csr.colidx, csr.values)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(wd).double(),
                                     torch.from_numpy(b).double(), stride=s, padding=p).numpy()
    assert np.abs(ref).max() < 2 ** 24
    assert np.array_equal(y.astype(np.float64), ref)


# ---------------------------------------------------------------- closed forms
def test_delta_filters_shift_input():
    C, H, W, K = 5, 7, 9, 3
    x = synthgen.make_input((2, C, H, W), 42)
    for ky in range(K):
        for kx in range(K):
            # F = C, filter f has one tap (c=f, ky, kx) = 1 -> out = input shifted, zero-filled
            rowptr = np.arange(C + 1, dtype=np.int32)
            colidx = np.array([(f * K + ky) * K + kx for f in range(C)], np.int32)
            y = oracle.conv_f32(x, C, K, 1, 1, rowptr, colidx, np.ones(C, np.float32))
            ref = np.zeros_like(x)
            dy, dx = ky - 1, kx - 1
            for oy in range(H):
                for ox in range(W):
                    iy, ix = oy + dy, ox + dx
                    if 0 <= iy < H and 0 <= ix < W:
                        ref[:, :, oy, ox] = x[:, :, iy, ix]
            assert np.array_equal(y, ref), (ky, kx)


def test_nnz_zero_gives_bias():
    x = synthgen.make_input((2, 3, 5, 5), 5)
    b = np.array([0.25, -1.5, 3.0, 0.0], np.float32)
    y = oracle.conv_f32(x, 4, 3, 1, 1, np.zeros(5, np.int32), np.zeros(0, np.int32),
                        np.zeros(0, np.float32), b)
    assert np.array_equal(y, np.broadcast_to(b[None, :, None, None], y.shape))


def test_linearity_disjoint_supports():
    F, C, K = 6, 4, 3
    csr = synthgen.make_csr(F, C, K, 0.4, 11, 12)
    x = synthgen.make_input((2, C, 8, 8), 13)
    # split each row's nonzeros alternately into two disjoint CSR matrices
    parts = [([0], [], []), ([0], [], [])]
    for f in range(F):
        for t, j in enumerate(range(csr.rowptr[f], csr.rowptr[f + 1])):
            rp, ci, vv = parts[t % 2]
            ci.append(csr.colidx[j]); vv.append(csr.values[j])
        for rp, ci, vv in parts:
            rp.append(len(ci))
    y = oracle.conv_f64(x, F, K, 1, 1, csr.rowptr, csr.colidx, csr.values)
    y1 = oracle.conv_f64(x, F, K, 1, 1, *map(np.array, parts[0]))
    y2 = oracle.conv_f64(x, F, K, 1, 1, *map(np.array, parts[1]))
    np.testing.assert_allclose(y, y1 + y2, rtol=1e-13, atol=1e-13)


def test_all_ones_interior_is_nine():
    # all-ones 3x3 on all-ones input -> every interior output is 9.
    x = np.ones((1, 1, 6, 6), np.float32)
    y = oracle.conv_f32(x, 1, 3, 1, 1, [0, 9], np.arange(9), np.ones(9, np.float32))
    assert np.all(y[0, 0, 1:-1, 1:-1] == 9.0)
    assert y[0, 0, 0, 0] == 4.0 and y[0, 0, 0, 2] == 6.0


# ---------------------------------------------------------------- fused block
@pytest.mark.parametrize("HW", [(8, 8), (9, 7), (5, 12)])
def test_fused_equals_torch_pool_of_relu(HW):
    H, W = HW
    F, C, K = 5, 4, 3
    csr = synthgen.make_csr(F, C, K, 0.3, 21, 22)
    x = synthgen.make_input((3, C, H, W), 23)
    b = synthgen.make_bias(F, 24)
    conv = oracle.conv_f32(x, F, K, 1, 1, csr.rowptr, csr.colidx, csr.values, b)
    ref, ridx = torch.nn.functional.max_pool2d(torch.relu(torch.from_numpy(conv)), 2, 2,
                                               return_indices=True)
    p, am = oracle.fused_f32(x, F, K, 1, 1, csr.rowptr, csr.colidx, csr.values, b)
    assert np.array_equal(bits(p), bits(ref.numpy()))
    assert np.array_equal(am, ridx.numpy().astype(np.int32))


def test_fused_all_negative_gives_zero():
    x = np.abs(synthgen.make_input((1, 2, 6, 6), 31)) + 0.5
    p, am = oracle.fused_f32(x, 3, 3, 1, 1, [0, 1, 2, 3], [4, 13, 4], [-1.0, -2.0, -0.5])
    assert np.all(p == 0.0) and np.all(np.signbit(p) == False)


# ---------------------------------------------------------------- queries & threads
def test_points_match_full():
    cfg = synthgen.CONFIGS["c1"]
    L = synthgen.make_layer(cfg)
    c = L.csr
    y = oracle.conv_f32(L.x, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values)
    rng = np.random.default_rng(0)
    pts = np.stack([rng.integers(0, s, 200) for s in y.shape], axis=1)
    v = oracle.conv_points_f32(L.x, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values, None, pts)
    assert np.array_equal(bits(v), bits(y[tuple(pts.T)]))
    b = synthgen.make_bias(cfg.F, 9)
    pf, amf = oracle.fused_f32(L.x, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values, b)
    pts2 = np.stack([rng.integers(0, s, 100) for s in pf.shape], axis=1)
    v2, a2 = oracle.fused_points_f32(L.x, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values, b, pts2)
    assert np.array_equal(bits(v2), bits(pf[tuple(pts2.T)]))
    assert np.array_equal(a2, amf[tuple(pts2.T)])


@pytest.mark.parametrize("name,N,stride,pad", [("c1", 1, 1, 1), ("c2", 1, 1, 1), ("c1", 2, 2, 0)])
def test_points_f64_vs_torch_conv2d(name, N, stride, pad):
    """oracle_conv_points_f64 (the FP64 tolerance reference of the full-size sampled GPU
    tests) against torch.nn.functional.conv2d in float64 on the densified filters (a
    library routine, PAPER.md L308-330 semantics), at sampled points incl. all borders:
    within 1e-12.  A dropped tap, a wrong (ky, kx) decode or a missing bias fails it."""
    cfg = synthgen.CONFIGS[name].with_batch(N)
    L = synthgen.make_layer(cfg)
    c = L.csr
    b = synthgen.make_bias(cfg.F, 77)
    wd = densify(cfg.F, cfg.C, cfg.K, c.rowptr, c.colidx, c.values)
    ref = torch.nn.functional.conv2d(torch.from_numpy(L.x).double(), torch.from_numpy(wd).double(),
                                     torch.from_numpy(b).double(), stride=stride, padding=pad).numpy()
    rng = np.random.default_rng(11)
    pts = np.stack([rng.integers(0, s, 500) for s in ref.shape], axis=1)
    edge = np.array([(n, f, yy, xx) for n in (0, ref.shape[0] - 1) for f in (0, ref.shape[1] - 1)
                     for yy in (0, ref.shape[2] - 1) for xx in (0, ref.shape[3] - 1)])
    pts = np.concatenate([pts, edge])
    v = oracle.conv_points_f64(L.x, cfg.F, cfg.K, stride, pad, c.rowptr, c.colidx, c.values, b, pts)
    assert v.dtype == np.float64
    assert np.max(np.abs(v - ref[tuple(pts.T)])) <= 1e-12


def test_thread_count_invariance():
    cfg = synthgen.CONFIGS["c1"].with_batch(3)
    L = synthgen.make_layer(cfg)
    c = L.csr
    y1 = oracle.conv_f32(L.x, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values, nthreads=1)
    y4 = oracle.conv_f32(L.x, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values, nthreads=5)
    assert np.array_equal(bits(y1), bits(y4))


def test_f32_ordered_within_contract_of_f64():
    # The north_star tolerance (1e-5 rel, 1e-4 abs) must hold between the two
    # oracle modes at the longest row lengths used (c4 at 50%: ~1152 terms/row).
    F, C, K = 4, 256, 3
    csr = synthgen.make_csr(F, C, K, 0.5, 51, 52)
    x = synthgen.make_input((2, C, 6, 6), 53)
    y32 = oracle.conv_f32(x, F, K, 1, 1, csr.rowptr, csr.colidx, csr.values)
    y64 = oracle.conv_f64(x, F, K, 1, 1, csr.rowptr, csr.colidx, csr.values)
    ok, worst = allclose_contract(y32, y64)
    assert ok, worst


# ---------------------------------------------------------------- CSR validation
def test_check_csr_errors():
    F, C, K = 2, 2, 3
    good = (np.array([0, 2, 3], np.int32), np.array([1, 5, 17], np.int32),
            np.array([1, 2, 3], np.float32))
    assert oracle.check_csr(F, C, K, *good) == 0
    bad = [
        (np.array([1, 2, 3]), good[1], good[2]),          # rowptr[0] != 0
        (np.array([0, 2, 2]), good[1], good[2]),          # rowptr[F] != nnz
        (np.array([0, 3, 2]), good[1][:2], good[2][:2]),  # decreasing
        (good[0], np.array([1, 5, 18]), good[2]),         # col out of range
        (good[0], np.array([5, 1, 17]), good[2]),         # unsorted
        (good[0], np.array([5, 5, 17]), good[2]),         # duplicate
        (good[0], np.array([-1, 5, 17]), good[2]),        # negative
        (good[0], good[1], np.array([1, np.nan, 3])),     # non-finite
    ]
    for b in bad:
        assert oracle.check_csr(F, C, K, *b) == -3, b


# ---------------------------------------------------------------- NEXT-3 block epilogue (reading R1)
def test_epilogue_residual_relu_matches_definition():
    """conv_ex = ReLU((conv + bias) + residual): the composition written out with numpy
    FP32 adds (IEEE RN, the same single rounding per step) and v > 0 ? v : +0."""
    cfg = synthgen.CONFIGS["c1"].with_batch(2)
    L = synthgen.make_layer(cfg)
    c = L.csr
    b = synthgen.make_bias(cfg.F, 99)
    res = synthgen.make_input((2, cfg.F, 16, 16), 98)
    args = (L.x, cfg.F, 3, 1, 1, c.rowptr, c.colidx, c.values, b)
    base = oracle.conv_f32(*args)
    for relu in (False, True):
        for r in (None, res):
            got = oracle.conv_ex_f32(*args, residual=r, relu=relu)
            want = base.copy() if r is None else (base + r).astype(np.float32)
            if relu:
                want = np.where(want > 0, want, np.float32(0.0)).astype(np.float32)
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_resnet_block_chain_vs_torch_float64():
    """A ResNet basic block composed from oracle layers agrees with the same block in
    float64 torch (dense conv2d of the densified filters) within the FP32 contract."""
    torch = pytest.importorskip("torch")
    C, H, W, N = 8, 9, 7, 2
    c1 = synthgen.make_csr(C, C, 3, 0.3, 501, 502)
    c2 = synthgen.make_csr(C, C, 3, 0.2, 503, 504)
    b1, b2 = synthgen.make_bias(C, 505), synthgen.make_bias(C, 506)
    x = synthgen.make_input((N, C, H, W), 507)
    y1 = oracle.conv_ex_f32(x, C, 3, 1, 1, c1.rowptr, c1.colidx, c1.values, b1, relu=True)
    y2 = oracle.conv_ex_f32(y1, C, 3, 1, 1, c2.rowptr, c2.colidx, c2.values, b2, residual=x, relu=True)
    w1 = torch.from_numpy(densify(C, C, 3, c1.rowptr, c1.colidx, c1.values)).double()
    w2 = torch.from_numpy(densify(C, C, 3, c2.rowptr, c2.colidx, c2.values)).double()
    xt = torch.from_numpy(x).double()
    t1 = torch.relu(torch.nn.functional.conv2d(xt, w1, torch.from_numpy(b1).double(), padding=1))
    t2 = torch.relu(torch.nn.functional.conv2d(t1, w2, torch.from_numpy(b2).double(), padding=1) + xt)
    err = np.abs(y2 - t2.numpy())
    assert (err <= 1e-4 + 1e-5 * np.abs(t2.numpy())).all(), err.max()


# ---------------------------------------------------------------- NEXT-2 resize (reading R2)
@pytest.mark.parametrize("hw", [(13, 17), (26, 34), (7, 9), (20, 11), (1, 1), (40, 3)])
def test_resize_bilinear_vs_torch_float64(hw):
    """Half-pixel bilinear resize == torch interpolate(mode='bilinear', align_corners=False)
    evaluated in float64, within FP32 rounding of the weights (inputs in [-1, 1))."""
    x = synthgen.make_input((2, 3, 13, 17), 31337)
    y = oracle.resize_bilinear_f32(x, *hw)
    t = torch.nn.functional.interpolate(torch.from_numpy(x).double(), size=hw, mode="bilinear",
                                        align_corners=False).numpy()
    assert np.abs(y - t).max() <= 4e-6


def test_resize_identity_and_constant():
    x = synthgen.make_input((1, 2, 9, 11), 4242)
    assert np.array_equal(oracle.resize_bilinear_f32(x, 9, 11).view(np.uint32), x.view(np.uint32))
    c = np.full((1, 1, 5, 6), 0.375, np.float32)
    for hw in [(10, 12), (3, 2), (17, 7)]:
        assert (oracle.resize_bilinear_f32(c, *hw) == np.float32(0.375)).all()
