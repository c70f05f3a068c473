"""Multi-GPU host logic of the RB online solver.

One process per GPU (torchrun); torch.distributed is the plumbing (NCCL on
GPUs, gloo in the CPU tests).  Nothing here computes any step of the method:

* query sharding -- the queries are independent units (PAPER.md:155-169 and
  260-279 solve one mu at a time), so they are split into contiguous shards
  with no collective on the data path; W and the offline blocks (PAPER.md:
  110-114 eq12c) are built once on the root rank and broadcast;
* slab partition -- the z-plane ranges of a mesh split for one huge system
  (the c5 layout), with the ghost planes a stencil of radius `ghost` needs.
"""
from __future__ import annotations


def query_shard(n_queries: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, stop) of rank's queries; shard sizes differ by at most 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(int(n_queries), world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def slab_partition(m: int, world: int, rank: int, ghost: int = 1) -> dict:
    """z-planes of rank's slab of an m^3 grid (interior planes 1..m): owned
    [z0, z1), stored [g0, g1) including up to `ghost` planes per side (clipped
    at the Dirichlet boundary), planes balanced to within one."""
    z0, z1 = query_shard(m, world, rank)
    z0, z1 = z0 + 1, z1 + 1
    return {"z0": z0, "z1": z1, "g0": max(1, z0 - ghost), "g1": min(m + 1, z1 + ghost),
            "owned": z1 - z0}


def broadcast_basis(W, ANq, fn, src: int = 0, group=None):
    """Broadcast W (N x n) and the offline blocks from `src` to every rank, in place
    (tensors must already have the right shape/dtype on the receiving ranks)."""
    import torch.distributed as dist
    for t in (W, ANq, fn):
        dist.broadcast(t, src, group=group)
    return W, ANq, fn


def gather_counts(its, status, group=None):
    """All-gather per-query iteration counts / statuses (int tensors of equal
    length on every rank) for the run's metrics; returns concatenated tensors."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out_i = [torch.empty_like(its) for _ in range(world)]
    out_s = [torch.empty_like(status) for _ in range(world)]
    dist.all_gather(out_i, its, group=group)
    dist.all_gather(out_s, status, group=group)
    return torch.cat(out_i), torch.cat(out_s)


def batch_order(mus, B: int):
    """Host-side batch scheduling: the query order that groups queries of similar
    coefficient contrast (max / min of the parameters, the spread of the diffusion
    coefficient) into the same batch of B lanes.  A batch runs until its slowest
    query converges (frozen lanes still stream through every pass), and the contrast
    is a cheap proxy for a query's RBCG iteration count (correlation ~0.6 on c1), so
    sorted batches waste fewer lane-iterations.  Every query's iterates are
    independent of its batch (DESIGN.md AMB-26): only the schedule changes.
    Returns a permutation of range(len(mus)), stable for equal contrast."""
    import numpy as np
    mus = np.asarray(mus, dtype=np.float64)
    if mus.ndim != 2 or B < 1:
        raise ValueError("mus must be (n_queries, P), B >= 1")
    lm = np.log(np.maximum(mus, np.finfo(np.float64).tiny))
    contrast = lm.max(axis=1) - lm.min(axis=1)
    return np.argsort(contrast, kind="stable")
