"""Host-side checks of the sharding plumbing (no GPU): slab partitioning, and DistTransport's
halo exchange / all_gather / any() over a world_size-2 gloo process group on CPU."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def test_make_slabs_tiles_volume():
    from paper_2410_08946_b200 import shard
    for D in (1, 2, 7, 768):
        for K in range(1, min(D, 8) + 1):
            s = shard.make_slabs(D, K)
            assert s[0].z0 == 0 and s[-1].z1 == D
            assert all(a.z1 == b.z0 for a, b in zip(s, s[1:]))
            assert all(x.z1 > x.z0 for x in s)
            assert all(x.e0 == max(0, x.z0 - 2) and x.e1 == min(D, x.z1 + 2) for x in s)
            assert all(x.zlo == x.z0 - x.e0 and x.zhi == x.z1 - x.e0 for x in s)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2410_08946_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tr = shard.DistTransport()
    lo = torch.full((6,), 10 * rank + 1, dtype=torch.int32)   # first plane -> rank-1
    hi = torch.full((6,), 10 * rank + 2, dtype=torch.int32)   # last plane -> rank+1
    below, above = tr.exchange([lo if rank > 0 else None], [hi if rank < world - 1 else None])
    g = tr.allgather([torch.arange(3, dtype=torch.int32) + 100 * rank])[0]
    a = tr.any([rank == 1])
    n = tr.allgather_i64([rank + 5])[0]
    q.put((rank, None if below[0] is None else below[0].tolist(), None if above[0] is None else above[0].tolist(),
           g.tolist(), a, n))
    dist.destroy_process_group()


def test_dist_transport_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    # rank 0 receives rank 1's first plane from above; rank 1 receives rank 0's last plane from below
    assert res[0][0] is None and res[0][1] == [11] * 6
    assert res[1][0] == [2] * 6 and res[1][1] is None
    for r in (0, 1):
        assert res[r][2] == [0, 1, 2, 100, 101, 102]
        assert res[r][3] is True
        assert res[r][4] == [5, 6]
