"""The seeded input generator (shared by both sides; holds no method arithmetic)."""
import numpy as np
import pytest

import synthgen


def test_splitmix64_reference_values():
    # SplitMix64 with state 0: published first outputs of the reference generator
    # (Steele, Lea & Flood 2014; java.util.SplittableRandom / Vigna's splitmix64.c).
    u = synthgen.splitmix64(0, np.arange(3, dtype=np.uint64))
    assert [int(v) for v in u] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


@pytest.mark.parametrize("name,nnz", [("c1", 461), ("c2", 7373), ("c3", 3686), ("c4_50", 294912),
                                      ("c4_80", 117965), ("c4_90", 58982), ("c4_95", 29491),
                                      ("c5", 22118)])
def test_config_nnz(name, nnz):
    cfg = synthgen.CONFIGS[name]
    assert cfg.nnz == nnz
    csr = synthgen.make_csr(cfg.F, cfg.C, cfg.K, cfg.density, synthgen.seed_of(cfg.k, 0),
                            synthgen.seed_of(cfg.k, 1))
    assert csr.nnz == nnz
    assert csr.rowptr[0] == 0 and csr.rowptr[-1] == nnz
    assert np.all(np.diff(csr.rowptr) >= 0)
    for f in range(cfg.F):
        seg = csr.colidx[csr.rowptr[f]:csr.rowptr[f + 1]]
        assert np.all(np.diff(seg) > 0)
    assert csr.colidx.min() >= 0 and csr.colidx.max() < cfg.C * cfg.K * cfg.K
    assert np.all(csr.values != 0) and np.all(np.abs(csr.values) <= 1)


def test_useful_flops_c2():
    assert synthgen.CONFIGS["c2"].useful_flops == 2 * 7373 * 32 * 56 * 56


def test_input_counter_based_and_chunk_invariant():
    a = synthgen.make_input((2, 3, 5, 7), 99, chunk=7)
    b = synthgen.make_input((2, 3, 5, 7), 99)
    assert np.array_equal(a, b)
    idx = np.array([0, 5, 100, 209])
    assert np.array_equal(synthgen.input_at(99, idx), b.reshape(-1)[idx])
    assert b.min() >= -1 and b.max() < 1
    # 24-bit grid: every value times 2^23 is an integer
    assert np.all((b.astype(np.float64) * 2 ** 23) % 1 == 0)


def test_integer_mode_ranges():
    csr = synthgen.make_csr(8, 8, 3, 0.5, 1, 2, integer=True)
    assert set(np.unique(csr.values).tolist()) <= {-4, -3, -2, -1, 1, 2, 3, 4}
    x = synthgen.make_input((1, 4, 6, 6), 3, integer=True)
    assert x.min() >= -4 and x.max() <= 4
    b = synthgen.make_bias(16, 4, integer=True)
    assert b.min() >= -2 and b.max() <= 2


def test_skewed_rows_mode():
    csr = synthgen.make_csr(64, 64, 3, 0.2, 5, 6, skew=1.5)
    counts = np.diff(csr.rowptr)
    assert csr.nnz == synthgen.nnz_for(64, 64, 3, 0.2)
    assert counts.max() / counts.mean() > 1.5


def test_deterministic():
    a = synthgen.make_layer(synthgen.CONFIGS["c1"])
    b = synthgen.make_layer(synthgen.CONFIGS["c1"])
    assert np.array_equal(a.csr.colidx, b.csr.colidx) and np.array_equal(a.x, b.x)
