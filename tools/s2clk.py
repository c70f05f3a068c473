"""Per-warp cycle accounting of k_smooth2 on c2 (instrumented build, -DRBS_CLK).

  RBS_NVCC_EXTRA="-DRBS_CLK [-DRBS_S2PIPE=1]" python tools/s2clk.py [--iters K]
Rebuilds librbs.so with the given flags (do not ship that build), runs K RBCG
iterations eagerly on the c2 batch and prints cycles per march step by warp
role: [issue, wait, sweep, work/out, barrier].
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1804_06363_b200 import build  # noqa: E402

build.build(force=True)
import paper_1804_06363_b200 as rbs  # noqa: E402
from synth import CONFIGS, query_set, train_set  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
c = CONFIGS["c2"]
s = rbs.Solver(c.dim, c.m, c.blocks)
s.build_greedy(train_set(c), c.n)
mus = query_set(c)[:c.B]
s.solve_batch(mus, tol=0.0, max_iter=2, want_a_n=False)
buf = (C.c_ulonglong * (148 * 16 * 6 + 148 * 3))()
lib = rbs.lib()
lib.rbs_debug_s2clk(buf)
out = s.solve_batch(mus, profile=1, tol=0.0, max_iter=a.iters, want_a_n=False)
lib.rbs_debug_s2clk(buf)
allv = np.frombuffer(buf, dtype=np.uint64).astype(np.float64)
v = allv[:148 * 16 * 6].reshape(148, 16, 6)
tt = allv[148 * 16 * 6:].reshape(148, 3)
m = c.m
nsx = (m + 31) // 32
nsy = max(1, 148 // nsx)
rps = max(8, (m + nsy - 1) // nsy)
nsy = (m + rps - 1) // rps
ncta = nsx * nsy
steps = (rps + 10) * (a.iters + 1)
v = v[:ncta] / steps
print(f"ctas {ncta} rows/seg {rps} steps/launch {rps + 10} launches {a.iters + 1}")
print("warp  issue   wait  sweep  work   barrier  total")
for w in range(16):
    r = v[:, w, :].mean(axis=0)
    print(f"{w:4d} " + " ".join(f"{x:6.0f}" for x in r[:5]) + f"  {r[:5].sum():6.0f}")
nc = ncta
t0 = tt[:nc, 0].min()
print("last launch, ns from first CTA entry: entry spread %.0f, loop start (min/max) %.0f/%.0f, exit (min/max) %.0f/%.0f"
      % (tt[:nc, 0].max() - t0, tt[:nc, 1].min() - t0, tt[:nc, 1].max() - t0, tt[:nc, 2].min() - t0, tt[:nc, 2].max() - t0))
print("profile (ms, launches):", {k: (round(x[0], 3), x[1]) for k, x in out["profile"].items()})
