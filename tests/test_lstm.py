"""NEXT-4: the sparse multilayer LSTM.

CPU: the oracle (oracle/lstm_oracle.c, reading R3) is pinned to torch.nn.LSTM in
float64 (a library routine with the same gate equations) and to the zero-weight case.
GPU (-m gpu): the CUDA wavefront and sequential schedules through the C-ABI agree
with each other bit for bit (every cell runs the same code on the same inputs, only
the launch grouping differs) and with the float64 oracle within the FP32 tolerance
derived in DESIGN.md (R3)."""
import numpy as np
import pytest

import oracle
import synthgen

torch = pytest.importorskip("torch")


def _torch_lstm(x, layers, D, H):
    L = len(layers)
    m = torch.nn.LSTM(D, H, num_layers=L).double()
    with torch.no_grad():
        for l, (rp, ci, vv, bb) in enumerate(layers):
            Dl = D if l == 0 else H
            G = np.zeros((4 * H, Dl + H))
            for r in range(4 * H):
                G[r, ci[rp[r]:rp[r + 1]]] = vv[rp[r]:rp[r + 1]]
            getattr(m, f"weight_ih_l{l}").copy_(torch.from_numpy(G[:, :Dl]))
            getattr(m, f"weight_hh_l{l}").copy_(torch.from_numpy(G[:, Dl:]))
            getattr(m, f"bias_ih_l{l}").copy_(torch.from_numpy(np.asarray(bb, np.float64)))
            getattr(m, f"bias_hh_l{l}").zero_()
        out, _ = m(torch.from_numpy(x).double())
    return out.numpy()


@pytest.mark.parametrize("L,D,H,T,B,d", [(1, 5, 4, 1, 1, 0.5), (2, 12, 8, 5, 3, 0.3), (3, 16, 16, 9, 2, 0.15),
                                         (4, 7, 6, 4, 5, 1.0)])
def test_oracle_matches_torch_lstm(L, D, H, T, B, d):
    layers, x = synthgen.make_lstm(L, D, H, d, T, B)
    h = oracle.lstm_f64(x, layers, H)
    assert np.abs(h - _torch_lstm(x, layers, D, H)).max() < 1e-12


def test_oracle_zero_weights_give_zero():
    L, D, H, T, B = 2, 6, 4, 3, 2
    layers = [(np.zeros(4 * H + 1, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32),
               np.zeros(4 * H, np.float32)) for _ in range(L)]
    x = synthgen.make_input((T, B, D), 11)
    assert (oracle.lstm_f64(x, layers, H) == 0.0).all()


def _gpu_case(L, D, H, T, B, d, batch_sample=None):
    from paper_2005_04091_b200.lstm import SEQUENTIAL, WAVEFRONT, SparseLSTM
    layers, x = synthgen.make_lstm(L, D, H, d, T, B)
    net = SparseLSTM(D, H, layers)
    xt = torch.from_numpy(x).cuda()
    hw = net(xt, WAVEFRONT).cpu().numpy()
    hs = net(xt, SEQUENTIAL).cpu().numpy()
    assert np.array_equal(hw.view(np.uint32), hs.view(np.uint32))
    cols = np.arange(B) if batch_sample is None else np.asarray(batch_sample)
    ref = oracle.lstm_f64(np.ascontiguousarray(x[:, cols, :]), layers, H)
    err = np.abs(hw[:, cols, :] - ref)
    assert (err <= 2e-5 + 1e-4 * np.abs(ref)).all(), err.max()
    net.close()


@pytest.mark.gpu
@pytest.mark.parametrize("L,D,H,T,B,d", [(1, 5, 4, 1, 1, 0.5), (2, 12, 8, 5, 3, 0.3), (4, 64, 48, 17, 70, 0.15),
                                         (3, 130, 96, 6, 33, 0.4)])
def test_gpu_lstm_parity(L, D, H, T, B, d):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _gpu_case(L, D, H, T, B, d)


@pytest.mark.gpu
@pytest.mark.parametrize("L,D,H,T,B,d", [(2, 100, 48, 7, 36, 0.2), (3, 130, 96, 6, 128, 0.4),
                                         (2, 64, 1024, 3, 64, 0.15)])
def test_gpu_lstm_staged_kernel(L, D, H, T, B, d, monkeypatch):
    """B >= 32 with 16-byte rows runs the z-staged kernel (chunks of 64 z rows in shared
    memory; D=100 makes a chunk straddle the [input ; h] boundary, B=36 a partial batch
    tile, B=128 two tiles, H=1024 with 2 cells the 16-warp CTA): parity with the oracle,
    and bitwise equality with the one-warp-per-unit kernel (same fma chains)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _gpu_case(L, D, H, T, B, d, batch_sample=None if B <= 40 else [0, B // 2, B - 1])
    from paper_2005_04091_b200.lstm import WAVEFRONT, SparseLSTM
    layers, x = synthgen.make_lstm(L, D, H, d, T, B)
    net = SparseLSTM(D, H, layers)
    xt = torch.from_numpy(x).cuda()
    h_staged = net(xt, WAVEFRONT).cpu().numpy()
    monkeypatch.setenv("SPCONV_LSTM_KERNEL", "rowwarp")  # knobs are read when a plan is created
    net_row = SparseLSTM(D, H, layers)
    h_row = net_row(xt, WAVEFRONT).cpu().numpy()
    assert np.array_equal(h_staged.view(np.uint32), h_row.view(np.uint32))
    net.close()
    net_row.close()


@pytest.mark.gpu
@pytest.mark.parametrize("wpc", ["8", "16"])
def test_gpu_lstm_staged_cta_sizes(wpc, monkeypatch):
    """8- and 16-warp CTAs of the staged kernel (SPCONV_LSTM_WPC) give the same bits."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_04091_b200.lstm import WAVEFRONT, SparseLSTM
    layers, x = synthgen.make_lstm(2, 70, 64, 0.2, 4, 40)
    xt = torch.from_numpy(x).cuda()
    monkeypatch.setenv("SPCONV_LSTM_KERNEL", "rowwarp")  # knobs are read when a plan is created
    net = SparseLSTM(70, 64, layers)
    ref = net(xt, WAVEFRONT).cpu().numpy()
    net.close()
    monkeypatch.delenv("SPCONV_LSTM_KERNEL")
    monkeypatch.setenv("SPCONV_LSTM_WPC", wpc)
    net = SparseLSTM(70, 64, layers)
    h = net(xt, WAVEFRONT).cpu().numpy()
    assert np.array_equal(h.view(np.uint32), ref.view(np.uint32))
    net.close()


@pytest.mark.gpu
def test_gpu_lstm_paper_size_sampled():
    """PAPER.md L510 sizes (4 layers, T=100, H=1024, 15% density), B=64, oracle on a
    sample of batch columns (they are independent)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _gpu_case(4, 1024, 1024, 100, 64, 0.15, batch_sample=[0, 31, 63])


@pytest.mark.gpu
def test_gpu_lstm_random_shapes(monkeypatch):
    """Seeded random LSTM shapes across the three cell kernels (lanes-over-nonzeros for
    B < 32, z-staged for B >= 32 with B % 4 == 0 and H % 8 == 0, one warp per unit
    otherwise): wavefront == sequential bitwise, staged == one-warp-per-unit bitwise,
    and the float64 oracle within the R3 tolerance on sampled batch columns."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_04091_b200.lstm import WAVEFRONT, SparseLSTM
    rng = np.random.default_rng(1510)
    for i in range(8):
        L = int(rng.integers(1, 4))
        D = int(rng.integers(1, 150))
        H = int(rng.choice([8, 16, 24, 40, 64, 13]))
        T = int(rng.integers(1, 8))
        B = int(rng.choice([1, 5, 32, 36, 44, 64, 66, 96]))
        d = float(rng.choice([0.05, 0.15, 0.5]))
        _gpu_case(L, D, H, T, B, d, batch_sample=None if B <= 8 else [0, B // 2, B - 1])
        layers, x = synthgen.make_lstm(L, D, H, d, T, B)
        net = SparseLSTM(D, H, layers)
        xt = torch.from_numpy(x).cuda()
        h_default = net(xt, WAVEFRONT).cpu().numpy()
        monkeypatch.setenv("SPCONV_LSTM_KERNEL", "rowwarp")  # read when a plan is created
        net_row = SparseLSTM(D, H, layers)
        h_row = net_row(xt, WAVEFRONT).cpu().numpy()
        net_row.close()
        monkeypatch.delenv("SPCONV_LSTM_KERNEL")
        if B >= 32:
            assert np.array_equal(h_default.view(np.uint32), h_row.view(np.uint32)), (i, L, D, H, T, B, d)
        net.close()
