"""Multi-GPU sharding of the FPE hot path (one process per GPU, torch.distributed).

The evaluation is embarrassingly parallel over points ("If the
number of evaluation points is high compared to the core count, the algorithm FPE is
embarrassingly parallel"), so the only exchange is ONE broadcast of the immutable
preconditioned buffer from the source rank (NCCL over NVLink/NVSwitch on GPUs, gloo in
the CPU tests).  Points are partitioned into contiguous shards; no collective touches
the data path.  Results are bitwise independent of the sharding (per-point purity).
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


def replicate(poly, src: int = 0, group=None, device: int | None = None):
    """Give every rank a handle of the source rank's preconditioned polynomial.

    Source: exports its flat device buffer; all ranks: one broadcast (NCCL), then
    fpe_poly_from_device_buffer on the received bytes (validated: magic/version/size).
    """
    import torch
    import torch.distributed as dist

    from . import Poly
    rank = dist.get_rank(group)
    if device is None:
        device = torch.cuda.current_device()
    dev = torch.device("cuda", device)
    buf = None
    if rank == src:
        buf = torch.empty(poly.nbytes, dtype=torch.uint8, device=dev)
        poly.export(buf.data_ptr(), poly.nbytes)
    buf = broadcast_buffer(buf, src=src, group=group, device=dev)
    torch.cuda.synchronize(dev)
    if rank == src:
        return poly
    return Poly.from_buffer(buf.data_ptr(), buf.numel(), device=device)


def evaluate_shard(poly, points_all, group=None, exps: bool = True):
    """Evaluate this rank's contiguous shard of a (replicated) point array on its GPU."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lo, hi = shard_range(len(points_all), rank, world)
    part = points_all[lo:hi]
    if isinstance(part, np.ndarray):
        part = torch.from_numpy(np.ascontiguousarray(part))
    part = part.to(torch.device("cuda", poly.device))
    v, e = poly.evaluate(part, exps=exps)
    return (lo, hi), v, e
