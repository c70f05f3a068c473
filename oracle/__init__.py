"""CPU fp64 oracle for the RB online solvers (Nguyen & Chen, arXiv:1804.06363).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module.
It shares no code with the CUDA product path (`paper_1804_06363_b200/`), and
neither imports the other; both take their seeded inputs from `synth/`.

The arithmetic lives in `oracle.c` (plain C, -O2 -ffp-contract=off); this file
is ctypes marshalling plus two convenience helpers that only compose oracle
calls.  Citations (PAPER.md line / equation / algorithm) are in oracle.c and
oracle.h.  Parity status of each function is listed in DESIGN.md ("Oracle
pins"); every function here is pinned by a `-m "not gpu"` test.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

SYM_RBGS, FWD_RBGS, JACOBI, FWD_LEX, SYM_LEX = 0, 1, 2, 3, 4
PRECOND_POST, PRECOND_SYM = 0, 1
BETA_FR, BETA_PR = 0, 1
STATUS = {0: "CONVERGED", 1: "MAXIT", 2: "REDUCED_NOT_SPD", 3: "CURVATURE", 4: "PRECOND",
          5: "NONFINITE"}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


class _Opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iter", C.c_int), ("smoother", C.c_int),
                ("sweeps", C.c_int), ("omega", C.c_double), ("delta", C.c_double),
                ("n_active", C.c_int), ("gamma", C.c_double), ("active_n", C.POINTER(C.c_int)),
                ("precond", C.c_int), ("beta_rule", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
    return _lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _blocks(blocks):
    b = list(blocks) + [1] * (3 - len(blocks))
    return (C.c_int * 3)(*b)


class Grid:
    """dim, m (interior nodes per axis), blocks (subdomains per axis) -- or faces: a
    general affine operator given by face coefficients faces[q][d][idx] (Q x dim x
    (m+1) m^(dim-1), layout in oracle.c; NEXT(4), DESIGN.md AMB-23)."""

    def __init__(self, dim: int, m: int, blocks=None, faces=None):
        self.dim, self.m = int(dim), int(m)
        self.N = self.m ** self.dim
        if faces is not None:
            nf = (self.m + 1) * self.m ** (self.dim - 1)
            self.faces = np.ascontiguousarray(faces, dtype=np.float64).reshape(-1, self.dim, nf)
            self.Q = self.faces.shape[0]
            self.blocks = None
            self._cb = (C.c_int * 3)(0, 0, 0)
        else:
            self.faces = None
            self.blocks = tuple(int(b) for b in blocks)
            assert len(self.blocks) == self.dim
            self.Q = int(np.prod(self.blocks))
            self._cb = _blocks(self.blocks)

    def _lib(self):
        """the oracle library with this grid's face operator bound (or none)."""
        L = lib()
        if self.faces is not None:
            L.or_set_faces(self.Q, _d(self.faces))
        else:
            L.or_set_faces(0, None)
        return L

    # -- operator / smoother ------------------------------------------------
    def apply_A(self, theta, x):
        theta = np.ascontiguousarray(theta, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.N)
        self._lib().or_apply_A(self.dim, C.c_int64(self.m), self._cb, _d(theta), _d(x), _d(y))
        return y

    def gs_halfsweep(self, theta, b, y, color):
        theta = np.ascontiguousarray(theta, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        y = np.array(y, dtype=np.float64, copy=True)
        self._lib().or_gs_halfsweep(self.dim, C.c_int64(self.m), self._cb, _d(theta), _d(b), _d(y),
                              int(color))
        return y

    def smooth(self, theta, b, y, kind=SYM_RBGS, sweeps=1, omega=1.0):
        theta = np.ascontiguousarray(theta, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        y = np.array(y, dtype=np.float64, copy=True)
        self._lib().or_smooth(self.dim, C.c_int64(self.m), self._cb, _d(theta), _d(b), _d(y),
                        int(kind), int(sweeps), C.c_double(omega))
        return y

    def dense_A(self, theta):
        """explicit matrix by applying the matrix-free operator to unit vectors (tiny grids)."""
        A = np.empty((self.N, self.N))
        e = np.zeros(self.N)
        for j in range(self.N):
            e[j] = 1.0
            A[:, j] = self.apply_A(theta, e)
            e[j] = 0.0
        return A

    # -- basis objects ------------------------------------------------------
    def offline_blocks(self, W):
        W = np.asfortranarray(W, dtype=np.float64)
        n = W.shape[1]
        ANq = np.empty((self.Q, n, n))
        fn = np.empty(n)
        self._lib().or_offline_blocks(self.dim, C.c_int64(self.m), self._cb, n, _d(W), _d(ANq), _d(fn))
        return ANq, fn

    # -- solvers ------------------------------------------------------------
    def _solve(self, fname, W, ANq, fn, mu, b, tol, max_iter, smoother, sweeps, omega, delta,
               n_active=0, gamma=0.0, precond=0, beta_rule=0):
        n = 0 if W is None else W.shape[1]
        Wf = np.asfortranarray(W, dtype=np.float64) if n else np.zeros((1, 1))
        ANq = np.ascontiguousarray(ANq, dtype=np.float64) if n else np.zeros(1)
        fn = np.ascontiguousarray(fn, dtype=np.float64) if n else np.zeros(1)
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        act = np.zeros(max_iter + 2, dtype=np.int32)
        o = _Opts(tol, max_iter, smoother, sweeps, omega, delta, int(n_active), float(gamma), _i(act),
                  int(precond), int(beta_rule))
        x = np.empty(self.N)
        its = C.c_int(0)
        hist = np.full(max_iter + 2, np.nan)
        a_n = np.full(max(n, 1), np.nan)
        trr = C.c_double(0)
        st = getattr(self._lib(), fname)(self.dim, C.c_int64(self.m), self._cb, n, _d(Wf), _d(ANq),
                                   _d(fn), _d(mu), _d(bb), C.byref(o), _d(x), C.byref(its),
                                   _d(hist), _d(a_n), C.byref(trr))
        k = its.value
        return dict(x=x, its=k, status=STATUS[st], hist=hist[:k + 1].copy(),
                    a_n=a_n[:n].copy(), true_relres=trr.value, active_n=act[:k].copy())

    def rbi(self, W, ANq, fn, mu, b=None, tol=1e-10, max_iter=500000, smoother=SYM_RBGS,
            sweeps=1, omega=1.0, delta=1e-12, n_active=0):
        return self._solve("or_rbi", W, ANq, fn, mu, b, tol, max_iter, smoother, sweeps,
                           omega, delta, n_active)

    def rbcg(self, W, ANq, fn, mu, b=None, tol=1e-10, max_iter=20000, smoother=SYM_RBGS,
             sweeps=1, omega=1.0, delta=1e-12, n_active=0, gamma=0.0, precond=PRECOND_POST,
             beta_rule=BETA_FR):
        """n_active: active RB dimension (0 = all columns); gamma > 0: the adaptive-n
        rule of PAPER.md:287 (the result's active_n[k] is the dimension of the k-th
        preconditioner application); precond: the paper's post-smoothed RBI (0) or the
        symmetric two-level RBI (1); beta_rule: as printed (0) or Polak-Ribiere (1)."""
        return self._solve("or_rbcg", W, ANq, fn, mu, b, tol, max_iter, smoother, sweeps,
                           omega, delta, n_active, gamma, precond, beta_rule)

    def precond_apply(self, W, ANq, mu, r, smoother=SYM_RBGS, sweeps=1, omega=1.0, precond=PRECOND_POST):
        """y = M^{-1} r, one application of the RBCG preconditioner (or_precond_apply)."""
        n = 0 if W is None else W.shape[1]
        Wf = np.asfortranarray(W, dtype=np.float64) if n else np.zeros((1, 1))
        A = np.ascontiguousarray(ANq, dtype=np.float64) if n else np.zeros(1)
        act = np.zeros(2, dtype=np.int32)
        o = _Opts(0.0, 1, smoother, sweeps, omega, 1e-12, 0, 0.0, _i(act), int(precond), 0)
        y = np.empty(self.N)
        r = np.ascontiguousarray(r, dtype=np.float64)
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        st = self._lib().or_precond_apply(self.dim, C.c_int64(self.m), self._cb, n, _d(Wf), _d(A), _d(mu),
                                          C.byref(o), _d(r), _d(y))
        assert st == 0
        return y

    def cg(self, mu, b=None, tol=1e-10, max_iter=100000):
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.N)
        its = C.c_int(0)
        st = self._lib().or_cg(self.dim, C.c_int64(self.m), self._cb, _d(mu), _d(bb), C.c_double(tol),
                         int(max_iter), _d(x), C.byref(its))
        return dict(x=x, its=its.value, status=STATUS[st])

    def greedy(self, mu_train, n_max, adaptive=True, snapshot_tol=1e-12, drop_tol=1e-10, phi_train=None,
               terms=None):
        """phi_train (nt, R) + terms (R, N): affine right-hand sides (or_set_greedy_rhs); the
        result's fnr is then (R, n) = W^T f_r."""
        mu_train = np.ascontiguousarray(mu_train, dtype=np.float64)
        nt = mu_train.shape[0]
        R = 0 if phi_train is None else int(np.shape(phi_train)[1])
        phi = np.ascontiguousarray(phi_train, dtype=np.float64) if R else None
        tm = np.ascontiguousarray(terms, dtype=np.float64) if R else None
        fnr = np.zeros((max(R, 1), n_max))
        self._lib().or_set_greedy_rhs(R, _d(phi), _d(tm), _d(fnr) if R else None)
        W = np.zeros((self.N, n_max), order="F")
        ANq = np.zeros((self.Q, n_max, n_max))
        fn = np.zeros(n_max)
        sel = np.full(n_max, -1, dtype=np.int32)
        ind = np.full(n_max, np.nan)
        its = np.zeros(n_max, dtype=np.int32)
        rej = C.c_int(0)
        n = self._lib().or_greedy(self.dim, C.c_int64(self.m), self._cb, nt, _d(mu_train), n_max,
                            int(adaptive), C.c_double(snapshot_tol), C.c_double(drop_tol),
                            _d(W), _d(ANq), _d(fn), _i(sel), _d(ind), _i(its), C.byref(rej))
        self._lib().or_set_greedy_rhs(0, None, None, None)
        out = dict(W=np.asfortranarray(W[:, :n]), ANq=ANq[:, :n, :n].copy(), fn=fn[:n].copy(),
                   selected=sel[:n].copy(), indicator=ind[:n].copy(), snap_iters=its[:n].copy(),
                   n_rejected=rej.value, n=n)
        if R:
            out["fnr"] = fnr[:, :n].copy()
        return out

    def basis_from_samples(self, mus, snapshot_tol=1e-12, drop_tol=1e-10):
        mus = np.ascontiguousarray(mus, dtype=np.float64)
        cnt = mus.shape[0]
        W = np.zeros((self.N, cnt), order="F")
        ANq = np.zeros((self.Q, cnt, cnt))
        fn = np.zeros(cnt)
        its = np.zeros(cnt, dtype=np.int32)
        rej = C.c_int(0)
        n = self._lib().or_basis_from_samples(self.dim, C.c_int64(self.m), self._cb, cnt, _d(mus),
                                        C.c_double(snapshot_tol), C.c_double(drop_tol), _d(W),
                                        _d(ANq), _d(fn), _i(its), C.byref(rej))
        return dict(W=np.asfortranarray(W[:, :n]), ANq=ANq[:, :n, :n].copy(), fn=fn[:n].copy(),
                    snap_iters=its[:n].copy(), n_rejected=rej.value, n=n)


# -- dense primitives --------------------------------------------------------
def adapt_n(rnorm_k, rnorm_k1, gamma, na, n_max):
    """The adaptive-n rule of PAPER.md:287 (or_adapt_n)."""
    return int(lib().or_adapt_n(C.c_double(rnorm_k), C.c_double(rnorm_k1), C.c_double(gamma),
                                int(na), int(n_max)))


def cholesky(A):
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    L = np.empty_like(A)
    piv = lib().or_cholesky(n, _d(A), _d(L))
    return L, piv


def chol_solve(L, b):
    L = np.ascontiguousarray(L, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty_like(b)
    lib().or_chol_solve(L.shape[0], _d(L), _d(b), _d(x))
    return x


def dot(x, y):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    lib().or_dot.restype = C.c_double
    return lib().or_dot(C.c_int64(x.size), _d(x), _d(y))


def mgs_append(W, v, drop_tol=1e-10):
    """returns (W_new, rejected)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    Nn = v.size
    n = 0 if W is None else W.shape[1]
    Wb = np.zeros((Nn, n + 1), order="F")
    if n:
        Wb[:, :n] = W
    rej = lib().or_mgs_append(C.c_int64(Nn), n, _d(Wb), _d(v), C.c_double(drop_tol))
    return (Wb if not rej else (W if n else np.zeros((Nn, 0), order="F"))), bool(rej)


def rb_solve(ANq, fn, mu):
    ANq = np.ascontiguousarray(ANq, dtype=np.float64)
    fn = np.ascontiguousarray(fn, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    n = fn.size
    a = np.empty(n)
    piv = lib().or_rb_solve(n, ANq.shape[0], _d(ANq), _d(fn), _d(mu), _d(a))
    return a, piv


# -- full-size test input recipe ---------------------------------------------
def interpolated_basis(dim, m, blocks, mu_train, n, m_coarse):
    """Oracle-built basis at a size where the oracle greedy is too slow
    (DESIGN.md "Input recipe"): greedy (algorithm3) on the coarse grid m_coarse,
    multilinear prolongation of its basis vectors to the fine grid (input
    generation only; (m+1) must be a multiple of (m_coarse+1)), then oracle MGS
     and oracle offline blocks (eq12c).  Returns (W, ANq, fn)."""
    from scipy.interpolate import RegularGridInterpolator
    assert (m + 1) % (m_coarse + 1) == 0
    gc = Grid(dim, m_coarse, blocks)
    res = gc.greedy(mu_train, n)
    hc, hf = 1.0 / (m_coarse + 1), 1.0 / (m + 1)
    axc = np.arange(m_coarse + 2) * hc
    fine = np.meshgrid(*[np.arange(1, m + 1) * hf] * dim, indexing="ij")
    pts = np.stack([f.reshape(-1, order="F") for f in fine], axis=1)  # x fastest
    W = None
    for j in range(res["n"]):
        v = np.zeros((m_coarse + 2,) * dim)
        inner = res["W"][:, j].reshape((m_coarse,) * dim, order="F")
        v[tuple(slice(1, m_coarse + 1) for _ in range(dim))] = inner
        vf = RegularGridInterpolator([axc] * dim, v)(pts)
        W, rej = mgs_append(W, vf)
    g = Grid(dim, m, blocks)
    ANq, fn = g.offline_blocks(W)
    return np.asfortranarray(W), ANq, fn


def _interp_axis(v, axis, m_c, m_f):
    """linear interpolation of nodal values along one axis from the coarse grid
    (m_c interior nodes, zero boundary) to the fine grid (m_f interior nodes); exact
    refinement: (m_f + 1) is a multiple of (m_c + 1).  Input generation only."""
    r = (m_f + 1) // (m_c + 1)
    v = np.moveaxis(v, axis, 0)
    pad = np.zeros((m_c + 2,) + v.shape[1:])
    pad[1:m_c + 1] = v
    I = np.arange(1, m_f + 1)
    lo, fr = I // r, (I % r) / r                                # coarse cell and fraction
    out = pad[lo] * (1.0 - fr)[(slice(None),) + (None,) * (v.ndim - 1)] + \
        pad[np.minimum(lo + 1, m_c + 1)] * fr[(slice(None),) + (None,) * (v.ndim - 1)]
    return np.moveaxis(out, 0, axis)


def offline_blocks_blas(g, W, threads=1):
    """A_{n,q} = W^T A_q W and f_n = W^T 1 (eq12c) with the oracle's
    matrix-free operator for A_q w_j (or_apply_A, one column at a time) and library
    products for W^T (A_q w_j) (numpy/BLAS; a library primitive as one step); (i <= j)
    mirrored as or_offline_blocks (O-3).  For full-size inputs, where or_offline_blocks'
    plain loops take minutes; pinned against it (tests/test_oracle_pins.py).  One
    column of A_q W at a time (memory: W plus `threads` columns); the C calls release
    the GIL, so columns run in `threads` threads."""
    from concurrent.futures import ThreadPoolExecutor
    W = np.asfortranarray(W, dtype=np.float64)
    n = W.shape[1]
    ANq = np.empty((g.Q, n, n))

    def col(qj):
        q, j = qj
        e = np.zeros(g.Q)
        e[q] = 1.0
        return q, j, W.T @ g.apply_A(e, W[:, j])

    jobs = [(q, j) for q in range(g.Q) for j in range(n)]
    with ThreadPoolExecutor(max(1, threads)) as ex:
        for q, j, c in ex.map(col, jobs):
            ANq[q][:, j] = c
    for q in range(g.Q):
        M = ANq[q]
        ANq[q] = np.triu(M) + np.triu(M, 1).T
    return ANq, W.T @ np.ones(W.shape[0])


def fullsize_basis(dim, m, blocks, mu_train, n, m_coarse, threads=1):
    """Full-size test input at the bench's RB dimension (DESIGN.md input recipe): greedy
    (algorithm3, or_greedy) on the coarse grid m_coarse, separable linear interpolation
    of its basis to the fine grid, orthonormalised in place (modified Gram-Schmidt with
    one re-orthogonalisation by library products: input generation, the span matters),
    offline blocks by offline_blocks_blas.  Memory: W plus a few columns.
    Returns (W, ANq, fn)."""
    gc = Grid(dim, m_coarse, blocks)
    res = gc.greedy(mu_train, n)
    assert res["n"] == n, res["n"]
    N = m ** dim
    W = np.empty((N, n), order="F")
    for j in range(n):
        v = res["W"][:, j].reshape((m_coarse,) * dim, order="F")   # axis 0 = x
        for ax in range(dim):
            v = _interp_axis(v, ax, m_coarse, m)
        w = v.reshape(-1, order="F")
        for _ in range(2):
            if j:
                w = w - W[:, :j] @ (W[:, :j].T @ w)
        W[:, j] = w / np.linalg.norm(w)
    ANq, fn = offline_blocks_blas(Grid(dim, m, blocks), W, threads)
    return W, ANq, fn
