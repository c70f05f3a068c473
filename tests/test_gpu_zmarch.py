"""GPU parity of the 3D z-plane marches (paper_1804_06363_b200/csrc/zmarch.cuh: k_cgz,
k_gsz, k_xrz fed by 4-D TMA tensor-map copies) -- RBCG Steps 5-7, 11 and the red-black
half-sweeps (eq8, 269-275 algorithm2) on grids that span several (x, y)
tiles, several z-segments and ragged tile edges in x, y and z, for every batch width
(B_pad 8 / 16 / 32).  Against the oracle (criteria of tests/test_gpu_parity.py) and against
the row-segment kernels they replace (RBS_DISABLE_V2 bit 16): the stencil is the same per
node, the uniform-block Gauss-Seidel update differs by rounding (AMB-27) and so does the
order of the per-CTA partial sums, so the two GPU paths agree to rounding and take the
same number of iterations."""
import os

import numpy as np
import pytest

from test_gpu_parity import compare, oracle_basis, oracle_refs, rbs  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def _solver_pair(rbs, dim, m, blocks, res, bits="65536"):
    z = rbs.Solver(dim, m, blocks).load_basis(res["W"], res["ANq"], res["fn"])
    old = os.environ.get("RBS_DISABLE_V2")
    os.environ["RBS_DISABLE_V2"] = bits             # read once at rbs_create
    try:
        r = rbs.Solver(dim, m, blocks).load_basis(res["W"], res["ANq"], res["fn"])
    finally:
        if old is None:
            del os.environ["RBS_DISABLE_V2"]
        else:
            os.environ["RBS_DISABLE_V2"] = old
    return z, r


# m = 37: B_pad 8 -> 2 x 5 tiles of 32 x 8 (ragged in x and y), 13 z-segments of 3 planes;
# B_pad 16 -> 3 x 5 tiles of 16 x 8; B_pad 32 -> 3 x 10 tiles of 16 x 4 (ragged y)
@pytest.mark.parametrize("m,blocks,n,B", [(37, (2, 2, 2), 12, 3), (37, (2, 3, 2), 16, 16),
                                          (29, (2, 2, 3), 10, 27), (8, (2, 2, 2), 6, 5)])
def test_zmarch_rbcg_matches_oracle_and_row_segments(orc, rbs, m, blocks, n, B):
    g, res = oracle_basis(orc, 3, m, blocks, n, 24, 5)
    z, r = _solver_pair(rbs, 3, m, blocks, res)
    mus = 0.1 * 100 ** np.random.default_rng(31 + B).random((B, g.Q))
    kw = dict(record_history=1, max_iter=20000)
    oz = z.solve_batch(mus, **kw)
    orow = r.solve_batch(mus, **kw)
    assert list(oz["status"]) == list(orow["status"])
    assert np.array_equal(oz["its"], orow["its"])
    Xz, Xr = oz["X"].cpu().numpy(), orow["X"].cpu().numpy()
    assert np.max(np.linalg.norm(Xz - Xr, axis=1) / np.linalg.norm(Xr, axis=1)) <= 1e-11
    sample = list(range(min(B, 4)))
    refs = oracle_refs(g, res["W"], res["ANq"], res["fn"], mus[sample], "rbcg", max_iter=20000)
    compare(dict(oz, X=oz["X"][sample], status=[oz["status"][i] for i in sample], its=oz["its"][sample],
                 a_n=oz["a_n"][sample], history=[oz["history"][i] for i in sample]),
            g, res["W"], res["ANq"], res["fn"], mus[sample], "rbcg", refs=refs)


@pytest.mark.parametrize("B", [8, 16, 32])
def test_zmarch_fixed_iterations_bitwise_node_values(orc, rbs, B):
    """Fixed-iteration RBCG (tol 0, 7 iterations) on a 41^3 grid: the z-march and the
    row-segment path agree to rounding at every lane (the only difference is the order
    of the CTA partial sums of sigma and y^T r)."""
    g, res = oracle_basis(orc, 3, 41, (2, 2, 2), 8, 20, 9)
    z, r = _solver_pair(rbs, 3, 41, (2, 2, 2), res)
    mus = 0.1 * 100 ** np.random.default_rng(B).random((B, g.Q))
    oz = z.solve_batch(mus, tol=0.0, max_iter=7)
    orow = r.solve_batch(mus, tol=0.0, max_iter=7)
    Xz, Xr = oz["X"].cpu().numpy(), orow["X"].cpu().numpy()
    assert np.max(np.abs(Xz - Xr)) <= 1e-12 * np.max(np.abs(Xr))
    ref = g.rbcg(res["W"], res["ANq"], res["fn"], mus[0], tol=0.0, max_iter=7)
    assert np.linalg.norm(Xz[0] - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])


@pytest.mark.parametrize("smoother,sweeps", [(0, 2), (1, 3)])
def test_zmarch_smoother_variants(orc, rbs, smoother, sweeps):
    """forward RB-GS with two sweeps and symmetric with three: the half-sweep sequence
    of k_gsz launches (colours, LAST epilogue) against the oracle."""
    g, res = oracle_basis(orc, 3, 19, (2, 2, 2), 8, 20, 3)
    s = rbs.Solver(3, 19, (2, 2, 2)).load_basis(res["W"], res["ANq"], res["fn"])
    mus = 0.1 * 100 ** np.random.default_rng(4).random((6, g.Q))
    out = s.solve_batch(mus, smoother=smoother, sweeps=sweeps, record_history=1)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbcg", smoother=smoother, sweeps=sweeps)


def test_zmarch_rbi(orc, rbs):
    """stand-alone RBI in 3D (the half-sweeps run as k_gsz; Step 2's residual keeps the
    projection pass) against the oracle."""
    g, res = oracle_basis(orc, 3, 15, (2, 2, 2), 10, 20, 2)
    s = rbs.Solver(3, 15, (2, 2, 2)).load_basis(res["W"], res["ANq"], res["fn"])
    mus = 0.1 * 100 ** np.random.default_rng(8).random((5, g.Q))
    out = s.solve_batch(mus, method=rbs.RBS_RBI, max_iter=500000, record_history=1)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbi", max_iter=500000)


@pytest.mark.parametrize("m,B", [(29, 16), (23, 5)])
def test_zmarch_faces_from_blocks(orc, rbs, m, B):
    """the face-coefficient instantiations of the z-plane marches (AMB-23: faces built
    from the thermal blocks reproduce the block operator) against the oracle, the
    block-operator z-march and the row-segment face kernels (RBS_DISABLE_V2 bit 17)"""
    from synth import cases
    blocks = (2, 2, 2)
    g, res = oracle_basis(orc, 3, m, blocks, 10, 24, 6)
    F = cases.faces_from_blocks(3, m, blocks)
    sf = rbs.Solver(3, m, faces=F).load_basis(res["W"], res["ANq"], res["fn"])
    sb = rbs.Solver(3, m, blocks).load_basis(res["W"], res["ANq"], res["fn"])
    old = os.environ.get("RBS_DISABLE_V2")
    os.environ["RBS_DISABLE_V2"] = "131072"
    try:
        sr = rbs.Solver(3, m, faces=F).load_basis(res["W"], res["ANq"], res["fn"])
    finally:
        if old is None:
            del os.environ["RBS_DISABLE_V2"]
        else:
            os.environ["RBS_DISABLE_V2"] = old
    mus = 0.1 * 100 ** np.random.default_rng(m + B).random((B, g.Q))
    of = sf.solve_batch(mus, record_history=1)
    ob = sb.solve_batch(mus)
    orr = sr.solve_batch(mus)
    assert np.all(np.abs(of["its"] - ob["its"]) <= 1)
    assert np.array_equal(of["its"], orr["its"])
    xf, xb, xr = (o["X"].cpu().numpy() for o in (of, ob, orr))
    assert np.linalg.norm(xf - xb) <= 1e-9 * np.linalg.norm(xb)
    assert np.linalg.norm(xf - xr) <= 1e-11 * np.linalg.norm(xr)
    sample = [0, B - 1]
    compare(dict(of, X=of["X"][sample], status=[of["status"][i] for i in sample], its=of["its"][sample],
                 a_n=of["a_n"][sample], history=[of["history"][i] for i in sample]),
            g, res["W"], res["ANq"], res["fn"], mus[sample], "rbcg")


@pytest.mark.parametrize("B", [5, 16, 27])
def test_zmarch_sym_precond_residual_projection(orc, rbs, B):
    """The symmetric two-level preconditioner's coarse correction W^T (r - A y1) on a 3D full
    grid: v = r - A y1 by k_xrz<RES> (z-plane march into the scratch vector) + the streamed
    k_wtr, against the flat k_proj<MODE_RESID> (RBS_DISABLE_V2 bit 19; same v per node, the
    W^T v partial sums in another order) and against the oracle's RB-PCG with the same
    preconditioner (NEXT(3)); m = 37 spans several ragged tiles and z-segments."""
    g, res = oracle_basis(orc, 3, 37, (2, 2, 2), 12, 24, 5)
    z, f = _solver_pair(rbs, 3, 37, (2, 2, 2), res, bits="524288")
    mus = 0.1 * 100 ** np.random.default_rng(71 + B).random((B, g.Q))
    kw = dict(record_history=1, max_iter=20000, precond=1)
    oz = z.solve_batch(mus, **kw)
    of = f.solve_batch(mus, **kw)
    assert all(st == "CONVERGED" for st in oz["status"]), oz["status"]
    assert np.max(np.abs(np.asarray(oz["its"]) - np.asarray(of["its"]))) <= 1
    Xz, Xf = oz["X"].cpu().numpy(), of["X"].cpu().numpy()
    assert np.max(np.linalg.norm(Xz - Xf, axis=1) / np.linalg.norm(Xf, axis=1)) <= 1e-9
    sample = list(range(min(B, 3)))
    compare(dict(oz, X=oz["X"][sample], status=[oz["status"][i] for i in sample], its=oz["its"][sample],
                 a_n=oz["a_n"][sample], history=[oz["history"][i] for i in sample]),
            g, res["W"], res["ANq"], res["fn"], mus[sample], "rbcg", max_iter=20000, precond=1)
    # fixed iterations (tol 0): the two GPU paths to rounding at every lane
    k = dict(tol=0.0, max_iter=6, precond=1)
    a, b = z.solve_batch(mus, **k)["X"].cpu().numpy(), f.solve_batch(mus, **k)["X"].cpu().numpy()
    assert np.max(np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)) <= 1e-12


@pytest.mark.parametrize("B", [5, 16])
def test_zmarch_rbi_residual_projection(orc, rbs, B):
    """Stand-alone RBI in 3D with Step 2's residual v = f - A x by k_xrz<RES> + k_wtr
    (PAPER.md:161-163): f = 1 (constant, no r tiles) against the oracle and the flat
    k_proj<MODE_RESID> (RBS_DISABLE_V2 bit 19); a given right-hand side (r tiles from
    rhs_dev) against the flat path in fixed-iteration mode."""
    import torch
    g, res = oracle_basis(orc, 3, 23, (2, 2, 2), 10, 20, 2)
    z, f = _solver_pair(rbs, 3, 23, (2, 2, 2), res, bits="524288")
    mus = 0.1 * 100 ** np.random.default_rng(90 + B).random((B, g.Q))
    kw = dict(method=rbs.RBS_RBI, max_iter=500000, record_history=1)
    oz = z.solve_batch(mus, **kw)
    of = f.solve_batch(mus, **kw)
    assert all(st == "CONVERGED" for st in oz["status"]), oz["status"]
    assert np.max(np.abs(np.asarray(oz["its"]) - np.asarray(of["its"]))) <= 1
    Xz, Xf = oz["X"].cpu().numpy(), of["X"].cpu().numpy()
    assert np.max(np.linalg.norm(Xz - Xf, axis=1) / np.linalg.norm(Xf, axis=1)) <= 1e-9
    sample = [0, B - 1]
    compare(dict(oz, X=oz["X"][sample], status=[oz["status"][i] for i in sample], its=oz["its"][sample],
                 a_n=oz["a_n"][sample], history=[oz["history"][i] for i in sample]),
            g, res["W"], res["ANq"], res["fn"], mus[sample], "rbi", max_iter=500000)
    rhs = torch.tensor(np.random.default_rng(3).standard_normal((B, g.N)), device="cuda")
    k = dict(method=rbs.RBS_RBI, tol=0.0, max_iter=8)
    a = z.solve_batch(mus, rhs=rhs, **k)["X"].cpu().numpy()
    b = f.solve_batch(mus, rhs=rhs, **k)["X"].cpu().numpy()
    assert np.max(np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)) <= 1e-12


@pytest.mark.parametrize("B,faces", [(5, False), (16, False), (27, False), (6, True)])
def test_zmarch_sym_presweep_from_zero(orc, rbs, B, faces):
    """The symmetric two-level preconditioner's pre-sweep y1 = S*(A, r, 0) (PAPER.md:161 in
    its pre+post-smoothed form, NEXT(3)): the first half-sweep from y = 0 as k_gsz<ZERO> (no
    fill, no y tiles: the sweep's colour gets D^{-1} r, the other colour and the frozen lanes
    0) against the k_fill_batch + half-sweep pair it replaces (RBS_DISABLE_V2 bit 20).  The
    same operations on the same operands: bitwise equal iterates, converged solves (queries
    freeze at different iterations) and fixed-iteration mode, and against the oracle."""
    from synth import cases
    m, blocks = 37, (2, 2, 2)
    g, res = oracle_basis(orc, 3, m, blocks, 12, 24, 5)
    kwf = dict(faces=cases.faces_from_blocks(3, m, blocks)) if faces else {}
    mk = (lambda: rbs.Solver(3, m, **kwf)) if faces else (lambda: rbs.Solver(3, m, blocks))
    z = mk().load_basis(res["W"], res["ANq"], res["fn"])
    old = os.environ.get("RBS_DISABLE_V2")
    os.environ["RBS_DISABLE_V2"] = "1048576"
    try:
        f = mk().load_basis(res["W"], res["ANq"], res["fn"])
    finally:
        if old is None:
            del os.environ["RBS_DISABLE_V2"]
        else:
            os.environ["RBS_DISABLE_V2"] = old
    mus = 0.1 * 100 ** np.random.default_rng(171 + B).random((B, g.Q))
    kw = dict(record_history=1, max_iter=20000, precond=1)
    oz = z.solve_batch(mus, **kw)
    of = f.solve_batch(mus, **kw)
    assert all(st == "CONVERGED" for st in oz["status"]), oz["status"]
    assert len(set(int(i) for i in oz["its"])) > 1 or B == 1     # lanes freeze at different iterations
    assert np.array_equal(oz["its"], of["its"])
    assert np.array_equal(oz["X"].cpu().numpy(), of["X"].cpu().numpy())
    for hz, hf in zip(oz["history"], of["history"]):
        assert np.array_equal(np.asarray(hz), np.asarray(hf))
    k = dict(tol=0.0, max_iter=6, precond=1)
    assert np.array_equal(z.solve_batch(mus, **k)["X"].cpu().numpy(), f.solve_batch(mus, **k)["X"].cpu().numpy())
    sample = [0, B - 1]
    compare(dict(oz, X=oz["X"][sample], status=[oz["status"][i] for i in sample], its=oz["its"][sample],
                 a_n=oz["a_n"][sample], history=[oz["history"][i] for i in sample]),
            g, res["W"], res["ANq"], res["fn"], mus[sample], "rbcg", max_iter=20000, precond=1)
