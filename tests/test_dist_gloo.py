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


def _worker_replicate(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_2211_06320_b200 as fpe
    import workloads
    from paper_2211_06320_b200.dist import gather_shards, replicate_buffer, shard_of
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = workloads.coefficients(5, d=(1 << 13) - 1)
    src = fpe.precondition_buffer(a) if rank == 0 else None     # only the source rank preconditions
    got = replicate_buffer(src, src=0).numpy()
    h = fpe.header_fields(got)
    # bench.py's cfg5 strong-scaling layout: each rank generates exactly its contiguous shard of the
    # seeded sequence; the shards reassemble the unsharded array
    n = 100003
    (lo, hi), _ = shard_of(np.empty(n))
    mine = workloads.points(5, hi - lo, start=lo)
    full = gather_shards(torch.from_numpy(mine.view(np.float64).reshape(-1, 2).copy()), n)
    q.put((rank, got.tobytes(), int(h["n_hull"]), lo, hi, full.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_replicate_buffer_and_shards(world):
    """replicate_buffer (the one broadcast of dist.replicate) with a host precondition_buffer on the source
    rank, shard_of + workloads' shard generation (bench.py --config 5) and gather_shards (verification):
    every rank holds the source's exact bytes, and the shards reassemble the unsharded point array."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_replicate, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    import paper_2211_06320_b200 as fpe
    import workloads
    ref = fpe.precondition_buffer(workloads.coefficients(5, d=(1 << 13) - 1)).tobytes()
    full = workloads.points(5, 100003).view(np.float64).tobytes()
    for r, (rank, b, nh, lo, hi, f) in enumerate(res):
        assert rank == r and b == ref and f == full
    assert res[0][3] == 0 and res[-1][4] == 100003
    assert all(res[i][4] == res[i + 1][3] for i in range(world - 1))


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
