"""Multi-GPU sharding of the FPE hot path (one process per GPU, torch.distributed).

The evaluation is embarrassingly parallel over points ("If the
number of evaluation points is high compared to the core count, the algorithm FPE is
embarrassingly parallel"), so the only exchange is ONE broadcast of the immutable
preconditioned buffer from the source rank (NCCL over NVLink/NVSwitch on GPUs, gloo in
the CPU tests).  Points are partitioned into contiguous shards; no collective touches
the data path.  Results are bitwise independent of the sharding (per-point purity), and
outputs stay sharded; gather_shards exists for verification only.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of ceil(n/world) points for `rank` (the last may be short)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    per = -(-n // world) if n > 0 else 0
    lo = min(n, rank * per)
    hi = min(n, lo + per)
    return lo, hi


def _rank_world(group=None) -> tuple[int, int]:
    import torch.distributed as dist
    if not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def broadcast_buffer(buf, src: int = 0, group=None, device=None):
    """Broadcast a flat uint8 buffer (torch tensor on `device`, or None off-source) from src.
    Returns the tensor on every rank.  Two collectives: the size, then the bytes."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    dev = device if device is not None else (buf.device if buf is not None else torch.device("cpu"))
    size = torch.tensor([buf.numel() if rank == src else 0], dtype=torch.int64, device=dev)
    dist.broadcast(size, src=src, group=group)
    if rank != src:
        buf = torch.empty(int(size.item()), dtype=torch.uint8, device=dev)
    dist.broadcast(buf, src=src, group=group)
    return buf


def replicate_buffer(poly_or_buffer, src: int = 0, group=None, device=None):
    """The source rank's flat preconditioned buffer on every rank (uint8 tensor on `device`).

    poly_or_buffer (source rank only): a Poly (its device buffer is exported) or a flat buffer (numpy
    uint8 from precondition_buffer, or a uint8 tensor).  Other ranks pass None."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    dev = torch.device(device) if device is not None else torch.device("cpu")
    buf = None
    if rank == src:
        x = poly_or_buffer
        if isinstance(x, np.ndarray):
            buf = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        elif isinstance(x, torch.Tensor):
            buf = x.to(dev)
        else:   # a Poly
            buf = torch.empty(x.nbytes, dtype=torch.uint8, device=dev)
            x.export(buf.data_ptr(), x.nbytes)
            if dev.type == "cuda":
                torch.cuda.synchronize(dev)
    return broadcast_buffer(buf, src=src, group=group, device=dev)


def replicate(poly, src: int = 0, group=None, device: int | None = None):
    """Give every rank a handle of the source rank's preconditioned polynomial.

    Source: exports its flat device buffer; all ranks: one broadcast (NCCL), then
    fpe_poly_from_device_buffer on the received bytes (validated: magic/version/size/sections).
    `poly` may also be a flat host buffer (precondition_buffer) on the source rank.
    """
    import torch
    import torch.distributed as dist

    from . import Poly
    rank = dist.get_rank(group)
    if device is None:
        device = torch.cuda.current_device()
    dev = torch.device("cuda", device)
    buf = replicate_buffer(poly if rank == src else None, src=src, group=group, device=dev)
    torch.cuda.synchronize(dev)
    if rank == src and isinstance(poly, Poly):
        return poly
    return Poly.from_buffer(buf.data_ptr(), buf.numel(), device=device)


def shard_of(points_all, group=None):
    """(lo, hi) and this rank's contiguous shard of a point array (numpy or tensor, any device)."""
    rank, world = _rank_world(group)
    lo, hi = shard_range(len(points_all), rank, world)
    return (lo, hi), points_all[lo:hi]


def evaluate_shard(poly, points_all, group=None, exps: bool = True):
    """Evaluate this rank's contiguous shard of a (replicated) point array on its GPU."""
    import torch
    (lo, hi), part = shard_of(points_all, group)
    if isinstance(part, np.ndarray):
        part = torch.from_numpy(np.ascontiguousarray(part))
    part = part.to(torch.device("cuda", poly.device))
    v, e = poly.evaluate(part, exps=exps)
    return (lo, hi), v, e


def gather_shards(x, n_total: int, group=None):
    """Verification only (untimed): the full length-n_total array of per-rank contiguous shards `x`
    (torch tensors, shard_range layout) on every rank.  Not part of the evaluation path."""
    import torch
    import torch.distributed as dist
    rank, world = _rank_world(group)
    if world == 1:
        return x
    per = shard_range(n_total, 0, world)[1]
    pad = torch.zeros((per,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[: x.shape[0]] = x
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = [parts[r][: shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0]] for r in range(world)]
    return torch.cat(out)
