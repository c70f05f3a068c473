"""Mesh slabs over ranks (c5-style): one 3D system split into z-slabs, one GPU per rank.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node G --master-addr 127.0.0.1 \\
        --master-port 29511 tools/slab_run.py --m 127 --n 16 --B 8

Rank 0 builds the basis with the GPU greedy on the full grid (offline, untimed),
broadcasts the offline blocks and scatters each rank the rows of its stored
planes; every rank joins the library's NCCL communicator (rbs_dist_init) and
solves the same queries (RBCG).  Rank 0 also solves the
unpartitioned system and checks that the gathered slab solution agrees; the
timed region is max-over-ranks CUDA-event time.  (The runs of this round had a
single GPU: the multi-rank path is exercised by tests/test_gpu_parity.py through
virtual slabs and a one-rank NCCL communicator.)
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_06363_b200 as rbs  # noqa: E402
from synth import loguniform_mu  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=127)
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--B", type=int, default=8)
ap.add_argument("--lo", type=float, default=0.01)
ap.add_argument("--hi", type=float, default=100.0)
a = ap.parse_args()
world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
m, blocks, P = a.m, (2, 2, 2), 8
N, plane = m ** 3, m * m
if rank == 0:
    full = rbs.Solver(3, m, blocks, device=local)
    gr = full.build_greedy(loguniform_mu(1005, 64, P, a.lo, a.hi), a.n, load=True)
    W = gr["W"].contiguous()
    n = gr["n"]
    meta = torch.tensor([n], device="cuda")
else:
    meta = torch.zeros(1, dtype=torch.int64, device="cuda")
dist.broadcast(meta, 0)
n = int(meta.item())
ANq = torch.tensor(gr["ANq"], device="cuda") if rank == 0 else torch.empty((P, n, n), dtype=torch.float64, device="cuda")
fn = torch.tensor(gr["fn"], device="cuda") if rank == 0 else torch.empty((n,), dtype=torch.float64, device="cuda")
dist.broadcast(ANq, 0)
dist.broadcast(fn, 0)
uid = [rbs.rbs_nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, 0)
s = rbs.Solver(3, m, blocks, device=local).dist_init(uid[0], world, rank, 3)
lr = s.local
# rows of the stored planes [g0, g1) of the full basis, from rank 0
rows = torch.empty((lr["n_stored"], n), dtype=torch.float64, device="cuda")
spans = [None] * world
dist.all_gather_object(spans, (lr["g0"], lr["g1"]))
if rank == 0:
    for r, (g0, g1) in enumerate(spans):
        blk = W[(g0 - 1) * plane:(g1 - 1) * plane].contiguous()
        if r == 0:
            rows.copy_(blk)
        else:
            dist.send(blk, r)
else:
    dist.recv(rows, 0)
s.load_basis(rows, ANq.cpu().numpy(), fn.cpu().numpy())
mus = loguniform_mu(2005, a.B, P, a.lo, a.hi)
s.solve_batch(mus)                     # warm-up (captures the iteration graph)
dist.barrier()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
out = s.solve_batch(mus)
e1.record()
torch.cuda.synchronize()
t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MAX)
parts = [None] * world
dist.all_gather_object(parts, out["X"].cpu().numpy())
if rank == 0:
    Xs = np.concatenate(parts, axis=1)
    ref = full.solve_batch(mus)
    Xf = ref["X"].cpu().numpy()
    err = float(np.abs(Xs - Xf).max() / np.abs(Xf).max())
    print(json.dumps({"ranks": world, "m": m, "N": N, "n": n, "B": a.B, "its": out["its"].tolist(),
                      "its_1gpu": ref["its"].tolist(), "max_rel_x_diff": err,
                      "ms_max_over_ranks": float(t.item()),
                      "queries_per_s": a.B / (float(t.item()) / 1e3)}))
dist.destroy_process_group()
