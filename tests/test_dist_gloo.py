"""Multi-process (world size 2, gloo, CPU) tests of the sharding path's host logic:
shard ranges partition the points, and the preconditioned flat buffer produced on the
source rank arrives byte-identical on the other rank and decodes to the same handle
contents (the single exchange of the distributed hot path)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_2211_06320_b200 as fpe
    import workloads
    from paper_2211_06320_b200.dist import broadcast_buffer, shard_range
    dist.init_process_group("gloo", rank=rank, world_size=world)
    buf = None
    if rank == 0:
        a = workloads.coefficients(3, d=(1 << 14) - 1)
        buf = torch.from_numpy(fpe.precondition_buffer(a))
    got = broadcast_buffer(buf, src=0)
    h = fpe.header_fields(got.numpy())
    lo, hi = shard_range(1000003, rank, world)
    q.put((rank, got.numpy().tobytes(), h["n_hull"], h["drop"], lo, hi))
    dist.barrier()
    dist.destroy_process_group()


def test_broadcast_and_shards_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, b0, nh0, d0, lo0, hi0), (r1, b1, nh1, d1, lo1, hi1) = res
    assert b0 == b1 and nh0 == nh1 and d0 == d1
    sys.path.insert(0, ROOT)
    import paper_2211_06320_b200 as fpe
    import workloads
    ref = fpe.precondition_buffer(workloads.coefficients(3, d=(1 << 14) - 1))
    assert ref.tobytes() == b0
    assert (lo0, hi0, lo1, hi1) == (0, 500002, 500002, 1000003)


def test_shard_range_partition():
    from paper_2211_06320_b200.dist import shard_range
    for n in (0, 1, 7, 1 << 20, 1000003):
        for w in (1, 2, 3, 4, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
