"""Multi-process host logic (query sharding, basis broadcast, slab partition) on
CPU with the gloo backend, world_size 2 -- the same calls bench.py makes over
NCCL on GPUs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_06363_b200.dist import (broadcast_basis, gather_counts, query_shard,
                                        slab_partition)


def test_query_shard_covers_and_balances():
    for nq in (0, 1, 7, 256, 1024, 1023):
        for world in (1, 2, 3, 4, 8):
            spans = [query_shard(nq, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nq
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_slab_partition_covers_planes():
    for m in (7, 63, 511):
        for world in (1, 2, 4, 8):
            parts = [slab_partition(m, world, r, ghost=3) for r in range(world)]
            assert parts[0]["z0"] == 1 and parts[-1]["z1"] == m + 1
            assert all(parts[i]["z1"] == parts[i + 1]["z0"] for i in range(world - 1))
            for p in parts:
                assert 1 <= p["g0"] <= p["z0"] and p["z1"] <= p["g1"] <= m + 1
                assert p["z0"] - p["g0"] <= 3 and p["g1"] - p["z1"] <= 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N, n, Q = 1000, 8, 4
        g = torch.Generator().manual_seed(7)
        if rank == 0:
            W = torch.randn(N, n, dtype=torch.float64, generator=g)
            A = torch.randn(Q, n, n, dtype=torch.float64, generator=g)
            f = torch.randn(n, dtype=torch.float64, generator=g)
        else:
            W = torch.zeros(N, n, dtype=torch.float64)
            A = torch.zeros(Q, n, n, dtype=torch.float64)
            f = torch.zeros(n, dtype=torch.float64)
        broadcast_basis(W, A, f, src=0)
        digest = float(W.sum() + A.sum() + f.sum())
        a, b = query_shard(10, world, rank)
        its = torch.arange(a, b, dtype=torch.int32) + 100
        st = torch.zeros(b - a, dtype=torch.int32) + rank
        allits, allst = gather_counts(its, st)
        q.put((rank, digest, allits.tolist(), allst.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_broadcast_and_gather_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == pytest.approx(res[1][1], rel=0, abs=0)      # bitwise identical basis
    for _, _, its, st in res:
        assert its == list(range(100, 110))
        assert st == [0] * 5 + [1] * 5


def test_batch_order_is_a_contrast_sorted_permutation():
    """the batch scheduler returns a permutation that sorts the queries by the spread of
    their log-parameters (stable), so equal queries keep their seeded order"""
    import numpy as np
    from paper_1804_06363_b200.dist import batch_order
    rng = np.random.default_rng(3)
    mus = 0.1 * 100 ** rng.random((50, 9))
    mus[7] = mus[3]
    p = batch_order(mus, 8)
    assert sorted(p.tolist()) == list(range(50))
    lm = np.log(mus[p])
    c = lm.max(1) - lm.min(1)
    assert np.all(np.diff(c) >= 0)
    assert p.tolist().index(3) < p.tolist().index(7)
    with pytest.raises(ValueError):
        batch_order(mus[0], 8)
