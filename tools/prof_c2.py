"""Profiling driver: one c2 batch (B=32, n=40) in eager profile mode.

  python tools/prof_c2.py --build PATH   # GPU greedy basis -> PATH (torch.save)
  python tools/prof_c2.py --load PATH [--iters K] [--config c2]
The --load run launches: offline-free basis load, setup, then K RBCG
iterations (tol = 0) with every kernel launched eagerly; used under ncu.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_06363_b200 as rbs  # noqa: E402
from synth import CONFIGS, query_set, train_set  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--build")
ap.add_argument("--load")
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--config", default="c2")
ap.add_argument("--method", default="rbcg")
a = ap.parse_args()
c = CONFIGS[a.config]
s = rbs.Solver(c.dim, c.m, c.blocks)
if a.build:
    gr = s.build_greedy(train_set(c), c.n, load=False)
    torch.save({"W": gr["W"].cpu(), "ANq": gr["ANq"], "fn": gr["fn"],
                "snap": gr["snap_iters"].tolist(), "sel": gr["selected"].tolist()}, a.build)
    print(json.dumps({"snap_iters": gr["snap_iters"].tolist(), "n": gr["n"]}))
if a.load:
    d = torch.load(a.load, weights_only=False)
    s.load_basis(d["W"], d["ANq"], d["fn"])
    mus = query_set(c)[:c.B]
    meth = rbs.RBS_RBCG if a.method == "rbcg" else rbs.RBS_RBI
    out = s.solve_batch(mus, profile=1, tol=0.0, max_iter=a.iters, method=meth, want_a_n=False)
    torch.cuda.synchronize()
    print(json.dumps({k: [round(v[0] / max(v[1], 1) * 1e3, 2), v[1]]
                      for k, v in out["profile"].items()}))
    if os.environ.get("PROF_GRAPH"):
        # graph-mode iteration time (the way bench.py runs one batch): fixed 200 iterations
        s.solve_batch(mus, tol=0.0, max_iter=50, method=meth, want_a_n=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        s.solve_batch(mus, tol=0.0, max_iter=200, method=meth, want_a_n=False)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"graph_us_per_iter": round(e0.elapsed_time(e1) * 1e3 / 200, 1)}))
