"""Problem definitions for general affine operators (NEXT(4), DESIGN.md AMB-23).

Face-coefficient operators and affine right-hand sides, shared by the oracle
side and the CUDA side as INPUTS: the thermal-block operator written as faces,
and the paper's Case 1 / Case 2 (Table 1) on a 7-point
finite-difference grid.  Nothing here is the paper's method (no residual,
projection, reduced solve, prolongation, smoothing or CG step): only the
coefficient fields, the source term and the Dirichlet lifting that define
A(theta) and f(mu).

Face layout (also in oracle.c and include/rbs.h): faces[q][d][idx], d = axis,
nf = (m+1) m^(dim-1) faces per axis; the face between nodes a and a+1 along d
(a = 0..m; nodes 0 and m+1 are Dirichlet nodes) has
  x: idx = a + (m+1)((J-1) + m(K-1))
  y: idx = (I-1) + m(a + (m+1)(K-1))
  z: idx = (I-1) + m((J-1) + m a).
The operator is A(theta) = (m+1)^2 K(theta), (K x)_P = sum_e kappa_e (x_P - x_P'),
kappa_e = sum_q theta_q faces[q][e]  (DESIGN.md AMB-3, AMB-23).
"""
from __future__ import annotations

import numpy as np


def n_faces(dim: int, m: int) -> int:
    return (m + 1) * m ** (dim - 1)


def _face_nodes(dim: int, m: int, d: int):
    """integer coordinates (full grid, 0..m+1) of the two nodes of every face along d,
    in idx order: returns (lo, hi), each an int array (nf, 3)."""
    a = np.arange(m + 1)
    i = np.arange(1, m + 1)
    one = np.array([1])
    if dim == 2:
        ks = one
    else:
        ks = i
    if d == 0:
        K, J, A = np.meshgrid(ks, i, a, indexing="ij")
        lo = np.stack([A, J, K], -1)
    elif d == 1:
        K, A, I = np.meshgrid(ks, a, i, indexing="ij")
        lo = np.stack([I, A, K], -1)
    else:
        A, J, I = np.meshgrid(a, i, i, indexing="ij")
        lo = np.stack([I, J, A], -1)
    lo = lo.reshape(-1, 3)
    hi = lo.copy()
    hi[:, d] += 1
    if dim == 2:
        lo[:, 2] = hi[:, 2] = 0
    return lo, hi


def faces_from_blocks(dim: int, m: int, blocks) -> np.ndarray:
    """The thermal-block operator as faces: the coefficient of a face is the mean of
    the cells sharing it (AMB-1), each cell in the block of its centre (AMB-2)."""
    p = list(blocks) + [1] * (3 - len(blocks))
    Q = int(np.prod(p[:dim]))

    def blk(c, pp):                     # cell index 0..m along an axis
        return ((2 * c + 1) * pp) // (2 * (m + 1))

    nf = n_faces(dim, m)
    F = np.zeros((Q, dim, nf))
    for d in range(dim):
        lo, _ = _face_nodes(dim, m, d)
        others = [ax for ax in range(dim) if ax != d]
        # cells sharing the face: along d the cell index is lo[d]; along the other
        # axes the cells lo-1 and lo (2^(dim-1) cells)
        offs = np.array(np.meshgrid(*[[-1, 0]] * (dim - 1), indexing="ij")).reshape(dim - 1, -1).T
        w = 1.0 / len(offs)
        for off in offs:
            c = np.zeros((nf, 3), dtype=np.int64)
            c[:, d] = lo[:, d]
            for k, ax in enumerate(others):
                c[:, ax] = lo[:, ax] + off[k]
            q = blk(c[:, 0], p[0]) + p[0] * blk(c[:, 1], p[1])
            if dim == 3:
                q = q + p[0] * p[1] * blk(c[:, 2], p[2])
            np.add.at(F[:, d, :], (q, np.arange(nf)), w)
    return F


def _coords(idx3, m):
    return idx3.astype(np.float64) / (m + 1)


def kappa_fields(case: int):
    """the coefficient fields of Table 1 as kappa = F_0 + mu_1 F_1:
    F_0 = 1, F_1 = r^2 (Case 1) or sin^2(20 pi (4(x-1/2)^2 + (y-1/2)^2 + (z-1/2)^2)) (Case 2,
    the unbalanced parenthesis read as SPEC.md:500 does, AMB-17)."""
    def one(x, y, z):
        return np.ones_like(x)

    if case == 1:
        def f1(x, y, z):
            return (x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2
    else:
        def f1(x, y, z):
            return np.sin(20 * np.pi * (4 * (x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2)) ** 2
    return [one, f1]


def faces_from_nodal(dim: int, m: int, fields) -> np.ndarray:
    """face coefficient = mean of the nodal field at the face's two nodes."""
    nf = n_faces(dim, m)
    F = np.zeros((len(fields), dim, nf))
    for d in range(dim):
        lo, hi = _face_nodes(dim, m, d)
        xl, xh = _coords(lo, m), _coords(hi, m)
        for q, f in enumerate(fields):
            F[q, d] = 0.5 * (f(*xl.T) + f(*xh.T))
    return F


def node_xyz(dim: int, m: int):
    """coordinates of the interior unknowns in the order P = (I-1) + m(J-1) + m^2(K-1)."""
    i = np.arange(1, m + 1) / (m + 1)
    if dim == 2:
        Y, X = np.meshgrid(i, i, indexing="ij")
        return X.ravel(), Y.ravel(), np.zeros(m * m)
    Z, Y, X = np.meshgrid(i, i, i, indexing="ij")
    return X.ravel(), Y.ravel(), Z.ravel()


def source(dim: int, m: int) -> np.ndarray:
    """3 pi^2 sin(pi x) sin(pi y) sin(pi z) (the sign read for an SPD system, AMB-17)."""
    x, y, z = node_xyz(dim, m)
    s = np.sin(np.pi * x) * np.sin(np.pi * y)
    return (3 * np.pi ** 2) * s * (np.sin(np.pi * z) if dim == 3 else 1.0)


def lifting(dim: int, m: int, F: np.ndarray, g) -> np.ndarray:
    """Dirichlet lifting of boundary data g for each operator term q:
    L_q[P] = (m+1)^2 sum over faces e of P with a boundary neighbour B of F_q[e] g(B),
    so that A(theta) u = f + sum_q theta_q L_q for u = g on the boundary."""
    Q, nf = F.shape[0], F.shape[2]
    L = np.zeros((Q, m ** dim))
    for d in range(dim):
        lo, hi = _face_nodes(dim, m, d)
        for side in (0, 1):          # boundary node at the low end (a = 0) or high end (a = m)
            sel = lo[:, d] == 0 if side == 0 else hi[:, d] == m + 1
            B = lo[sel] if side == 0 else hi[sel]
            P = hi[sel] if side == 0 else lo[sel]
            gb = g(*_coords(B, m).T)
            pidx = (P[:, 0] - 1) + m * (P[:, 1] - 1) + (m * m * (P[:, 2] - 1) if dim == 3 else 0)
            for q in range(Q):
                np.add.at(L[q], pidx, F[q, d, sel] * gb)
    return L * float(m + 1) ** 2


def case_problem(case: int, m: int, dim: int = 3):
    """Case 1 / Case 2 of Table 1 on m^dim interior nodes.  Returns dict(faces (2, dim, nf),
    terms (R, N): the right-hand-side terms, theta(mu) -> (2,), phi(mu) -> (R,), domain)."""
    F = faces_from_nodal(dim, m, kappa_fields(case))
    f = source(dim, m)
    if case == 1:
        return dict(faces=F, terms=f[None, :], domain=[(0.0, 1.0)],
                    theta=lambda mu: np.array([1.0, mu[0]]),
                    phi=lambda mu: np.array([1.0]))

    def ga(x, y, z):
        return np.cos(10 * np.pi * (4 * (x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2))

    def gb(x, y, z):
        return np.cos(10 * np.pi * (x + y + z))

    La, Lb = lifting(dim, m, F, ga), lifting(dim, m, F, gb)
    terms = np.stack([f, La[0], Lb[0], La[1], Lb[1]])
    return dict(faces=F, terms=terms, domain=[(0.0, 2.0), (0.0, 1.0)],
                theta=lambda mu: np.array([1.0, mu[0]]),
                phi=lambda mu: np.array([1.0, 1.0 - mu[1], mu[1], mu[0] * (1.0 - mu[1]), mu[0] * mu[1]]))


def case_params(case: int, count: int, seed: int) -> np.ndarray:
    """uniform samples of the parameter domain D (AMB-18)."""
    rng = np.random.default_rng(seed)
    dom = [(0.0, 1.0)] if case == 1 else [(0.0, 2.0), (0.0, 1.0)]
    return np.stack([lo + (hi - lo) * rng.random(count) for lo, hi in dom], axis=1)
