"""Multi-process host logic of the batch-sharded driver,
world_size 2 over gloo: sharding, CSR broadcast, output all-gather (on CPU with an oracle
stand-in layer, and -m gpu with two ranks sharing cuda:0 running the CUDA kernels).

The per-rank layer is injected (``layer_factory``); here it is the CPU oracle, so the
test checks the distribution logic (every image computed exactly once, gathered in
order, filters identical on every rank) — the CUDA forward itself is covered by the
-m gpu parity tests and by bench.py under torchrun on the box.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle  # noqa: E402
import synthgen  # noqa: E402
from paper_2005_04091_b200.parallel import (ShardedSparseConv2d, broadcast_csr,  # noqa: E402
                                            gather_output, shard_bounds)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _OracleLayer:
    """CPU stand-in for SparseConv2d (test-only)."""

    def __init__(self, cfg, rp, ci, vv, b):
        self.cfg = cfg
        self.args = (cfg.F, cfg.K, cfg.stride, cfg.pad, rp.numpy(), ci.numpy(), vv.numpy(),
                     None if b is None else b.numpy())

    def __call__(self, x):
        return torch.from_numpy(oracle.conv_f32(x.numpy(), *self.args))

    def fused_relu_maxpool(self, x):
        p, a = oracle.fused_f32(x.numpy(), *self.args)
        return torch.from_numpy(p), torch.from_numpy(a)


def _worker(rank, world, port, n_total, fused, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synthgen.CONFIGS["c1"].with_batch(n_total)
        L = synthgen.make_layer(cfg)
        bias = synthgen.make_bias(cfg.F, synthgen.seed_of(cfg.k, 3))
        src = (L.csr.rowptr, L.csr.colidx, L.csr.values, bias) if rank == 0 else (None, None, None, None)
        layer = ShardedSparseConv2d(cfg.F, *src, device=torch.device("cpu"),
                                    layer_factory=lambda rp, ci, vv, b: _OracleLayer(cfg, rp, ci, vv, b))
        b0, b1 = layer.local_shard(n_total)
        x_shard = torch.from_numpy(L.x[b0:b1].copy())
        out = layer.forward_gather(x_shard, n_total, fused=fused)
        if rank == 0:
            if fused:
                q.put((out[0].numpy(), out[1].numpy()))
            else:
                q.put(out.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_total,fused", [(4, False), (5, False), (3, True)])
def test_sharded_forward_gather_equals_single_process(n_total, fused):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_total, fused, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = synthgen.CONFIGS["c1"].with_batch(n_total)
    L = synthgen.make_layer(cfg)
    bias = synthgen.make_bias(cfg.F, synthgen.seed_of(cfg.k, 3))
    args = (L.x, cfg.F, cfg.K, cfg.stride, cfg.pad, L.csr.rowptr, L.csr.colidx, L.csr.values, bias)
    if fused:
        rp, ra = oracle.fused_f32(*args)
        assert np.array_equal(got[0].view(np.uint32), rp.view(np.uint32))
        assert np.array_equal(got[1], ra)
    else:
        ref = oracle.conv_f32(*args)
        assert got.shape == ref.shape
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def _bcast_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synthgen.CONFIGS["c2"]
        L = synthgen.make_layer(cfg, with_input=False)
        if rank == 0:
            rp, ci, vv, b = broadcast_csr(L.csr.rowptr, L.csr.colidx, L.csr.values, None, cfg.F, "cpu")
        else:
            rp, ci, vv, b = broadcast_csr(None, None, None, None, cfg.F, "cpu")
        q.put((rank, rp.numpy(), ci.numpy(), vv.numpy(), b))
        # uneven gather: 3 images over 2 ranks
        y = torch.full((shard_bounds(3, world, rank)[1] - shard_bounds(3, world, rank)[0], 2), float(rank))
        g = gather_output(y, 3)
        q.put((rank, g.numpy()))
    finally:
        dist.destroy_process_group()


def test_broadcast_csr_and_uneven_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bcast_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    items = [q.get(timeout=120) for _ in range(4)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    L = synthgen.make_layer(synthgen.CONFIGS["c2"], with_input=False)
    csr_items = [it for it in items if len(it) == 5]
    gath = [it for it in items if len(it) == 2]
    assert len(csr_items) == 2 and len(gath) == 2
    for _, rp, ci, vv, b in csr_items:
        assert np.array_equal(rp, L.csr.rowptr)
        assert np.array_equal(ci, L.csr.colidx)
        assert np.array_equal(vv.view(np.uint32), L.csr.values.view(np.uint32))
        assert b is None
    for _, g in gath:
        # rank 0 owns images [0, 2), rank 1 owns [2, 3)
        assert np.array_equal(g[:, 0], np.array([0.0, 0.0, 1.0], np.float32))


@pytest.mark.parametrize("n,world", [(0, 1), (7, 1), (7, 2), (8, 4), (3, 8), (256, 8)])
def test_shard_bounds_partition(n, world):
    seen = []
    for r in range(world):
        b, e = shard_bounds(n, world, r)
        assert 0 <= b <= e <= n
        seen.extend(range(b, e))
    assert seen == list(range(n))
    sizes = [shard_bounds(n, world, r)[1] - shard_bounds(n, world, r)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def _gpu_worker(rank, world, port, n_total, q):
    """Two ranks sharing cuda:0 (gloo moves the CUDA tensors): CSR broadcast from rank 0
    as device tensors -> spconv_create from device pointers -> each rank's batch shard
    through the CUDA kernel -> all-gather.  The NCCL path on a multi-GPU box is the same
    code with backend "nccl" and one device per rank."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2005_04091_b200 import SparseConv2d
        cfg = synthgen.CONFIGS["c2"].with_batch(n_total)
        L = synthgen.make_layer(cfg)
        bias = synthgen.make_bias(cfg.F, synthgen.seed_of(cfg.k, 3))
        src = (L.csr.rowptr, L.csr.colidx, L.csr.values, bias) if rank == 0 else (None, None, None, None)
        dev = torch.device("cuda", 0)
        layer = ShardedSparseConv2d(cfg.F, *src, device=dev,
                                    layer_factory=lambda rp, ci, vv, b: SparseConv2d(
                                        cfg.C, cfg.H, cfg.W, cfg.F, 3, 1, 1, rp, ci, vv, b, device=0))
        b0, b1 = layer.local_shard(n_total)
        xs = torch.from_numpy(L.x[b0:b1].copy()).to(dev)
        y = layer.forward(xs)
        full = gather_output(y.cpu(), n_total)  # gloo gathers host copies
        p, am = layer.forward(xs, fused=True)
        fp = gather_output(p.cpu(), n_total)
        fa = gather_output(am.cpu(), n_total)
        if rank == 0:
            q.put((full.numpy(), fp.numpy(), fa.numpy()))
        layer.layer.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_match_single_process():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n_total = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    y, fp, fa = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    cfg = synthgen.CONFIGS["c2"].with_batch(n_total)
    L = synthgen.make_layer(cfg)
    bias = synthgen.make_bias(cfg.F, synthgen.seed_of(cfg.k, 3))
    args = (L.x, cfg.F, cfg.K, cfg.stride, cfg.pad, L.csr.rowptr, L.csr.colidx, L.csr.values, bias)
    assert np.array_equal(y.view(np.uint32), oracle.conv_f32(*args).view(np.uint32))
    rp, ra = oracle.fused_f32(*args)
    assert np.array_equal(fp.view(np.uint32), rp.view(np.uint32)) and np.array_equal(fa, ra)
