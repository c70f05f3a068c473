"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family of the library on tiny inputs (the 2D row marches, the 3D row-segment
passes, the flat kernels, Jacobi, the NEXT(3) variants, virtual slabs, the GPU greedy).

    compute-sanitizer --tool racecheck --error-exitcode 1 python tools/sanitize.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_06363_b200 as rbs  # noqa: E402


def basis(N, n, seed):
    return np.linalg.qr(np.random.default_rng(seed).standard_normal((N, n)))[0]


def run():
    rng = np.random.default_rng(1)
    for dim, m, blocks, n, B in [(2, 40, (3, 3), 12, 32), (2, 21, (2, 2), 8, 5), (3, 11, (2, 2, 2), 8, 16)]:
        N = m ** dim
        Q = int(np.prod(blocks))
        s = rbs.Solver(dim, m, blocks).load_basis(basis(N, n, m))      # offline blocks on the device
        mus = 0.1 * 100 ** rng.random((B, Q))
        for kw in (dict(), dict(method=rbs.RBS_RBI, max_iter=40, tol=0.0), dict(smoother=1),
                   dict(smoother=2, omega=0.8), dict(precond=1), dict(beta_rule=1), dict(n_active=4, gamma=5.0)):
            out = s.solve_batch(mus, max_iter=kw.pop("max_iter", 60), record_history=1, **kw)
            print(dim, m, B, kw, out["status"][:2], int(out["its"].max()), flush=True)
        if dim == 3:
            s.set_slabs(2)
            out = s.solve_batch(mus[:4], max_iter=20)
            print("slabs", out["status"][:2], flush=True)
    g = rbs.Solver(2, 21, (2, 2))
    gr = g.build_greedy(0.1 * 100 ** rng.random((12, 4)), 4)
    print("greedy", gr["n"], list(gr["selected"]), flush=True)


if __name__ == "__main__":
    run()
    print("sanitize: done")
