"""Batch-sharded multi-GPU path over NCCL: two ranks, one
GPU each, CSR broadcast from rank 0, per-rank forward through the CUDA kernels, output
all-gather -- the gathered batch must equal the 1-GPU output bitwise (images are
independent: PAPER.md L335 ``conv.parallelize(n)``).  Skips below 2 GPUs (the round-end
box has one; the gloo tests cover the host logic on CPU)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthgen  # noqa: E402
from tests._util import bits  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, n_total, fused, q):
    import torch.distributed as dist

    from paper_2005_04091_b200 import SparseConv2d
    from paper_2005_04091_b200.parallel import ShardedSparseConv2d
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        cfg = synthgen.CONFIGS[name].with_batch(n_total)
        L = synthgen.make_layer(cfg)
        bias = synthgen.make_bias(cfg.F, synthgen.seed_of(cfg.k, 3))
        src = (L.csr.rowptr, L.csr.colidx, L.csr.values, bias) if rank == 0 else (None, None, None, None)
        sh = ShardedSparseConv2d(cfg.F, *src, device=dev,
                                 layer_factory=lambda rp, ci, vv, b: SparseConv2d(
                                     cfg.C, cfg.H, cfg.W, cfg.F, cfg.K, cfg.stride, cfg.pad, rp, ci, vv, b,
                                     device=rank))
        b0, b1 = sh.local_shard(n_total)
        x = torch.from_numpy(L.x[b0:b1]).to(dev)
        out = sh.forward_gather(x, n_total, fused)
        torch.cuda.synchronize()
        if rank == 0:
            full = SparseConv2d(cfg.C, cfg.H, cfg.W, cfg.F, cfg.K, cfg.stride, cfg.pad, L.csr.rowptr,
                                L.csr.colidx, L.csr.values, bias, device=0)
            xf = torch.from_numpy(L.x).to(dev)
            if fused:
                p1, a1 = full.fused_relu_maxpool(xf)
                ok = np.array_equal(bits(out[0].cpu().numpy()), bits(p1.cpu().numpy())) and \
                    np.array_equal(out[1].cpu().numpy(), a1.cpu().numpy())
            else:
                ok = np.array_equal(bits(out.cpu().numpy()), bits(full(xf).cpu().numpy()))
            q.put(ok)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,n_total,fused", [("c2", 7, False), ("c3", 6, True)])
def test_two_rank_nccl_gather_equals_one_gpu(name, n_total, fused):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, n_total, fused, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True
