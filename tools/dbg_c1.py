import os, sys, subprocess
code = r'''
import numpy as np, sys
sys.path.insert(0, ".")
import oracle, paper_1804_06363_b200 as rbs
from synth import CONFIGS, query_set, train_set
c = CONFIGS["c1"]
g = oracle.Grid(c.dim, c.m, c.blocks)
res = g.greedy(train_set(c), c.n)
s = rbs.Solver(c.dim, c.m, c.blocks).load_basis(res["W"], res["ANq"], res["fn"])
mus = query_set(c)
for meth in (rbs.RBS_RBCG, rbs.RBS_RBI):
    out = s.solve_batch(mus, method=meth, max_iter=20000 if meth else 500000)
    X = out["X"].cpu().numpy()
    ref = (g.rbcg if meth else g.rbi)(res["W"], res["ANq"], res["fn"], mus[0])
    print("meth", meth, out["status"][:2], out["its"][:3], ref["its"], np.linalg.norm(X[0]-ref["x"])/np.linalg.norm(ref["x"]))
'''
for mask in [0]:
    env = dict(os.environ, RBS_DISABLE_V2=str(mask))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    print("mask", mask, "rc", r.returncode, r.stdout.strip()[-400:], r.stderr.strip()[-300:])
