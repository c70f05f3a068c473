"""Independent test-side references used to PIN the oracle (not copies of it).

* `fem_p1_2d`: P1 finite-element stiffness on the structured right-triangle
  mesh with piecewise-constant kappa per cell (each square cell split along a
  diagonal), assembled element by element from barycentric gradients.  For
  these meshes this equals the cell-averaged 5-point system (DESIGN.md AMB-1;
  PAPER.md:319 uses P1 FEM).
* `cellwise_fd`: cell-by-cell assembly of the cell-averaged stencil: every
  cell scatters kappa_cell / 2^(d-1) to each of its axis edges.  A different
  indexing route than the oracle's node-by-node gather.
* `laplacian_eig`: textbook eigenpairs of the 5/7-point Dirichlet Laplacian.
* `sgs_rb_apply`: symmetric red-black Gauss-Seidel from zero as explicit
  triangular solves in the red-black ordering (textbook SGS preconditioner).
Kappa of a cell comes from the *geometric* location of its centre.
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def _cell_kappa(dim, m, blocks, mu):
    """kappa per cell (a,b[,c]) in 0..m, from the block containing its centre."""
    h = 1.0 / (m + 1)
    centers = (np.arange(m + 1) + 0.5) * h
    idx = [np.floor(centers * p).astype(int) for p in blocks]
    if dim == 2:
        q = idx[0][:, None] + blocks[0] * idx[1][None, :]
    else:
        q = (idx[0][:, None, None] + blocks[0] * idx[1][None, :, None]
             + blocks[0] * blocks[1] * idx[2][None, None, :])
    return np.asarray(mu)[q]  # indexed [a, b(, c)]


def _node_id(dim, m):
    """full-grid node (I,J[,K]) -> unknown index, -1 on the boundary."""
    shape = (m + 2,) * dim
    nid = -np.ones(shape, dtype=np.int64)
    inner = np.arange(m ** dim).reshape((m,) * dim, order="F")  # [i,j,k] = i + m j + m^2 k
    sl = tuple(slice(1, m + 1) for _ in range(dim))
    nid[sl] = inner  # x fastest (Fortran order over (I,J,K))
    return nid


def fem_p1_2d(m, blocks, mu, diag="main"):
    """h^-2-free P1 stiffness K (N x N sparse) on interior nodes."""
    h = 1.0 / (m + 1)
    kap = _cell_kappa(2, m, blocks, mu)
    nid = _node_id(2, m)
    rows, cols, vals = [], [], []
    for a in range(m + 1):
        for b in range(m + 1):
            c = [(a, b), (a + 1, b), (a + 1, b + 1), (a, b + 1)]
            tris = [(c[0], c[1], c[2]), (c[0], c[2], c[3])] if diag == "main" else \
                   [(c[0], c[1], c[3]), (c[1], c[2], c[3])]
            for tri in tris:
                X = np.array([[p[0] * h, p[1] * h] for p in tri])
                T = np.array([X[1] - X[0], X[2] - X[0]]).T  # 2x2
                area = 0.5 * abs(np.linalg.det(T))
                # gradients of barycentric functions
                Ginv = np.linalg.inv(T)           # maps x - X0 to (l1, l2)
                g = np.vstack([-Ginv.sum(axis=0), Ginv[0], Ginv[1]])
                Ke = kap[a, b] * area * (g @ g.T)
                for i in range(3):
                    for j in range(3):
                        I, J = nid[tri[i]], nid[tri[j]]
                        if I >= 0 and J >= 0:
                            rows.append(I); cols.append(J); vals.append(Ke[i, j])
    N = m * m
    return sp.csr_matrix((vals, (rows, cols)), shape=(N, N))


def fem_load_2d(m):
    """consistent P1 load of f = 1: integral of each interior hat function."""
    h = 1.0 / (m + 1)
    return np.full(m * m, h * h)


def cellwise_fd(dim, m, blocks, mu):
    """(m+1)^2 * sum_cells sum_edges w kappa_cell (e_P - e_P')(e_P - e_P')^T."""
    kap = _cell_kappa(dim, m, blocks, mu)
    nid = _node_id(dim, m)
    w = 0.5 if dim == 2 else 0.25
    rows, cols, vals = [], [], []
    for cell in itertools.product(range(m + 1), repeat=dim):
        k = w * kap[cell]
        for axis in range(dim):
            others = [d for d in range(dim) if d != axis]
            for offs in itertools.product((0, 1), repeat=dim - 1):
                p0 = list(cell)
                for d, o in zip(others, offs):
                    p0[d] += o
                p1 = list(p0)
                p1[axis] += 1
                I, J = nid[tuple(p0)], nid[tuple(p1)]
                for (u, v, s) in ((I, I, 1.0), (J, J, 1.0), (I, J, -1.0), (J, I, -1.0)):
                    if u >= 0 and v >= 0:
                        rows.append(u); cols.append(v); vals.append(s * k)
    N = m ** dim
    return (m + 1) ** 2 * sp.csr_matrix((vals, (rows, cols)), shape=(N, N))


def laplacian_eig(dim, m, ks):
    """eigenpair (lambda, v) of the unit-coefficient (m+1)^2-scaled Laplacian."""
    h = 1.0 / (m + 1)
    grids = np.meshgrid(*[np.arange(1, m + 1)] * dim, indexing="ij")
    v = np.ones_like(grids[0], dtype=float)
    lam = 0.0
    for g, k in zip(grids, ks):
        v = v * np.sin(k * np.pi * g * h)
        lam += 4.0 * np.sin(k * np.pi * h / 2) ** 2
    lam /= h * h
    return lam, v.reshape(-1, order="F")  # x fastest


def red_black_order(dim, m):
    grids = np.meshgrid(*[np.arange(1, m + 1)] * dim, indexing="ij")
    par = (sum(grids) % 2).reshape(-1, order="F")
    idx = np.arange(m ** dim)
    return np.concatenate([idx[par == 0], idx[par == 1]])


def sgs_rb_apply(A, order, r):
    """y = S_sym(A, r, 0): forward GS then backward GS in the given ordering."""
    Ap = A[order][:, order].tocsr()
    rp = r[order]
    Lw = sp.tril(Ap, format="csr")
    Up = sp.triu(Ap, format="csr")
    y1 = spla.spsolve_triangular(Lw, rp, lower=True)
    y = y1 + spla.spsolve_triangular(Up, rp - Ap @ y1, lower=False)
    out = np.empty_like(r)
    out[order] = y
    return out
