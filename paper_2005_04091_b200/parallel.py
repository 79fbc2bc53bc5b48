"""Batch-sharded multi-GPU driver, one process per GPU over
torch.distributed (NCCL on B200s; gloo for the CPU tests of the host logic).

Images are independent units (``conv.parallelize(n)`` makes the
batch loop the parallel one), so the batch is split into contiguous shards,
the filters are replicated, and the only collectives are:

  * ``broadcast_csr``: rank ``src`` broadcasts rowptr/colidx/values/bias once per
    plan (a7, "broadcast CSR + bias (once)");
  * ``gather_output``: an all-gather of the per-rank output shards into the
    full-batch NCHW tensor (batch-major, so each shard is a contiguous slice).

There is no collective inside the forward itself.
"""
from __future__ import annotations

import contextlib

import torch
import torch.distributed as dist


def _nvtx(name):
    """NVTX range around a collective (SURVEY.md §5 tracing); a no-op where unavailable."""
    try:
        return torch.cuda.nvtx.range(name)
    except Exception:  # pragma: no cover - torch without NVTX
        return contextlib.nullcontext()


def shard_bounds(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) shard of ``n_total`` images for ``rank`` (first ranks take
    the remainder)."""
    if world < 1 or not 0 <= rank < world or n_total < 0:
        raise ValueError("bad shard request")
    base, rem = divmod(n_total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def broadcast_csr(rowptr, colidx, values, bias, F: int, device, src: int = 0):
    """Broadcast the CSR filters (and optional bias) from ``src``; returns tensors on ``device``.

    Non-source ranks may pass None for the arrays; ``F`` must agree everywhere."""
    with _nvtx("spconv.broadcast_csr"):
        return _broadcast_csr(rowptr, colidx, values, bias, F, device, src)


def _broadcast_csr(rowptr, colidx, values, bias, F: int, device, src: int):
    rank = dist.get_rank()
    meta = torch.zeros(2, dtype=torch.int64, device=device)
    if rank == src:
        meta[0] = int(len(colidx))
        meta[1] = 0 if bias is None else 1
    dist.broadcast(meta, src)
    nnz, has_bias = int(meta[0]), bool(meta[1])

    def _t(a, n, dt):
        if rank == src:
            return torch.as_tensor(a, dtype=dt).to(device).contiguous()
        return torch.empty(n, dtype=dt, device=device)

    rp = _t(rowptr, F + 1, torch.int32)
    ci = _t(colidx, nnz, torch.int32)
    vv = _t(values, nnz, torch.float32)
    dist.broadcast(rp, src)
    if nnz:
        dist.broadcast(ci, src)
        dist.broadcast(vv, src)
    b = None
    if has_bias:
        b = _t(bias, F, torch.float32)
        dist.broadcast(b, src)
    return rp, ci, vv, b


def gather_output(y_shard: torch.Tensor, n_total: int) -> torch.Tensor:
    """All-gather per-rank output shards (shard_bounds layout) into the full batch."""
    with _nvtx("spconv.gather_output"):
        return _gather_output(y_shard, n_total)


def _gather_output(y_shard: torch.Tensor, n_total: int) -> torch.Tensor:
    world = dist.get_world_size()
    sizes = [shard_bounds(n_total, world, r) for r in range(world)]
    counts = [e - b for b, e in sizes]
    m = max(counts)
    per = y_shard.shape[1:]
    if all(c == m for c in counts) and hasattr(dist, "all_gather_into_tensor") and \
            dist.get_backend() == "nccl":
        out = torch.empty((n_total, *per), dtype=y_shard.dtype, device=y_shard.device)
        dist.all_gather_into_tensor(out, y_shard.contiguous())
        return out
    pad = torch.zeros((m, *per), dtype=y_shard.dtype, device=y_shard.device)
    pad[: y_shard.shape[0]] = y_shard
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


class ShardedSparseConv2d:
    """One SparseConv2d plan per rank on its own GPU; ``forward`` runs the local shard.

    ``layer_factory(rowptr, colidx, values, bias)`` builds the per-rank layer (the CUDA
    SparseConv2d in production); it is injectable so the host logic can be tested with
    gloo on CPU.
    """

    def __init__(self, F: int, rowptr, colidx, values, bias, device, layer_factory, src: int = 0):
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device
        rp, ci, vv, b = broadcast_csr(rowptr, colidx, values, bias, F, device, src)
        self.layer = layer_factory(rp, ci, vv, b)

    def local_shard(self, n_total: int) -> tuple[int, int]:
        return shard_bounds(n_total, self.world, self.rank)

    def forward(self, x_shard, fused: bool = False):
        if fused:
            return self.layer.fused_relu_maxpool(x_shard)
        return self.layer(x_shard)

    def forward_gather(self, x_shard, n_total: int, fused: bool = False):
        y = self.forward(x_shard, fused)
        if fused:
            return gather_output(y[0], n_total), gather_output(y[1], n_total)
        return gather_output(y, n_total)
