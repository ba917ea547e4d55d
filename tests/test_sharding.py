"""Host-side multi-rank logic on CPU: world_size-2 gloo processes shard sessions disjointly
and completely, and reduce step times with MAX (the bench's multi-GPU timing rule)."""

from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2511_02036_b200.sharding import session_seeds, shard_range


def test_shard_range_partitions_exactly():
    for n in (0, 1, 7, 64, 65):
        for world in (1, 2, 3, 4, 8):
            got = [shard_range(n, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [hi - lo for lo, hi in got]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2511_02036_b200.sharding import max_over_ranks, session_seeds, sum_over_ranks

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seeds = session_seeds(5000, 64, world, rank)
    t = max_over_ranks(10.0 + rank)
    n = sum_over_ranks(len(seeds))
    q.put((rank, seeds, t, n))
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_max_timing():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    seeds = out[0][1] + out[1][1]
    assert seeds == list(range(5000, 5064))
    assert set(out[0][1]).isdisjoint(out[1][1])
    assert out[0][2] == out[1][2] == 11.0
    assert out[0][3] == out[1][3] == 64
