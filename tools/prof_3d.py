"""Profiling driver for the flat 3D passes: thermal blocks 2x2x2 on M^3 (default 127), B = 16,
GPU greedy n = 20 from 64 training mu, then K RBCG iterations eagerly (tol = 0).
python tools/prof_3d.py [--m 127] [--iters 2] [--faces]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_06363_b200 as rbs  # noqa: E402
from synth import cases  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=127)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--faces", action="store_true")
ap.add_argument("--n", type=int, default=20)
ap.add_argument("--ntrain", type=int, default=64)
ap.add_argument("--random-basis", action="store_true",
                help="random orthonormal W (timing only: fixed-iteration solves, no greedy build)")
ap.add_argument("--B", type=int, default=16)
ap.add_argument("--precond", type=int, default=0, help="1: symmetric two-level preconditioner")
ap.add_argument("--rbi", action="store_true", help="stand-alone RBI instead of RBCG")
ap.add_argument("--prof-only", action="store_true", help="skip the graph-mode timing (ncu captures)")
a = ap.parse_args()
blocks = (2, 2, 2)
rng = np.random.default_rng(5)
tr = 0.1 * 100 ** rng.random((a.ntrain, 8))
if a.faces:
    s = rbs.Solver(3, a.m, faces=cases.faces_from_blocks(3, a.m, blocks))
else:
    s = rbs.Solver(3, a.m, blocks)
if a.random_basis:
    g = torch.Generator(device="cuda").manual_seed(1)
    W = torch.randn(a.m ** 3, a.n, device="cuda", dtype=torch.float64, generator=g)
    W, _ = torch.linalg.qr(W)
    s.load_basis(W)
    del W
elif os.environ.get("PROF3D_BASIS") and os.path.exists(os.environ["PROF3D_BASIS"]):
    d = torch.load(os.environ["PROF3D_BASIS"], weights_only=False)
    s.load_basis(d["W"], d["ANq"], d["fn"])
else:
    gr = s.build_greedy(tr, a.n)
    if os.environ.get("PROF3D_BASIS"):
        torch.save({"W": gr["W"].cpu(), "ANq": gr["ANq"], "fn": gr["fn"]}, os.environ["PROF3D_BASIS"])
mus = 0.1 * 100 ** rng.random((a.B, 8))
mkw = dict(method=rbs.RBS_RBI) if a.rbi else {}
torch.cuda.nvtx.range_push("solve")      # ncu --nvtx --nvtx-include "solve/" captures only this
out = s.solve_batch(mus, profile=1, tol=0.0, max_iter=a.iters, want_a_n=False, precond=a.precond, **mkw)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
prof = {k: [round(v[0] / max(v[1], 1) * 1e3, 2), v[1]] for k, v in out["profile"].items() if v[1]}
if a.prof_only:
    print(json.dumps(prof))
    sys.exit(0)
# graph-mode iteration time (the way bench.py runs): a fixed 200-iteration solve
s.solve_batch(mus, tol=0.0, max_iter=50, want_a_n=False, precond=a.precond, **mkw)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
s.solve_batch(mus, tol=0.0, max_iter=200, want_a_n=False, precond=a.precond, **mkw)
e1.record()
torch.cuda.synchronize()
prof["graph_us_per_iter"] = round(e0.elapsed_time(e1) * 1e3 / 200, 1)
print(json.dumps(prof))
