"""Tiny solves for compute-sanitizer (memcheck / racecheck / synccheck): a 2D row-march
RBCG + RBI and a 3D z-plane-march RBCG (block and face operators) on small grids with random
orthonormal bases (fixed 4 iterations)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1804_06363_b200 as rbs  # noqa: E402
from synth import cases  # noqa: E402


def basis(N, n, seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((N, n)))
    return q


rng = np.random.default_rng(1)
s2 = rbs.Solver(2, 37, (3, 3)).load_basis(basis(37 * 37, 12, 2))
mus = 0.1 * 100 ** rng.random((8, 9))
for meth in (rbs.RBS_RBCG, rbs.RBS_RBI):
    s2.solve_batch(mus, method=meth, tol=0.0, max_iter=4)
for kw in (dict(blocks=(2, 2, 2)), dict(faces=cases.faces_from_blocks(3, 21, (2, 2, 2)))):
    s3 = rbs.Solver(3, 21, **kw).load_basis(basis(21 ** 3, 8, 3))
    s3.solve_batch(0.1 * 100 ** rng.random((16, 8)), tol=0.0, max_iter=4)
torch.cuda.synchronize()
print("sanitize_small ok")
