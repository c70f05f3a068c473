"""GPU parity on the edges the main parity suite leaves out (VERDICT r1 "weak" 2):
breakdown status codes (CURVATURE, NONFINITE), the smallest grids (m = 1, 2, 3, 7 in
2D and 3D), single-query batches, and batch-composition invariance.  Oracle = the
CPU reference (oracle/); criteria as tests/test_gpu_parity.py."""
import numpy as np
import pytest

from test_gpu_parity import compare, oracle_basis, rbs  # noqa: F401  (fixture)
from synth import CONFIGS, query_set

pytestmark = pytest.mark.gpu


def _small2d(orc):
    # the oracle pins' small 2D problem: 15^2, 2x2 blocks, greedy n = 6 from 40 seeded mu
    g = orc.Grid(2, 15, (2, 2))
    tr = 0.1 * 100 ** np.random.default_rng(7).random((40, 4))
    return g, tr, g.greedy(tr, 6)


def test_curvature_breakdown(orc, rbs):
    """A block coefficient of the wrong sign with A_n(mu) still SPD: the oracle stops with
    CURVATURE (p^T A p <= 0, AMB-11) after one iteration; the GPU must too, while the
    other queries of the batch converge."""
    g, tr, res = _small2d(orc)
    bad = np.array([4.2701543811162175, -2.406109733991851, 0.16842629880036922, 6.70980228318393])
    An = np.einsum("q,qij->ij", bad, res["ANq"])
    assert np.linalg.eigvalsh(An).min() > 0          # the reduced matrix is SPD
    mus = np.vstack([tr[3], bad, tr[5]])
    s = rbs.Solver(2, 15, (2, 2)).load_basis(res["W"], res["ANq"], res["fn"])
    out = s.solve_batch(mus, record_history=1)
    ref = g.rbcg(res["W"], res["ANq"], res["fn"], bad)
    assert ref["status"] == "CURVATURE"
    assert out["status"] == ["CONVERGED", "CURVATURE", "CONVERGED"]
    assert out["its"][1] == ref["its"]
    compare(dict(out, X=out["X"][[0, 2]], status=[out["status"][0], out["status"][2]], its=out["its"][[0, 2]],
                 a_n=out["a_n"][[0, 2]], history=[out["history"][0], out["history"][2]]),
            g, res["W"], res["ANq"], res["fn"], mus[[0, 2]], "rbcg")


@pytest.mark.parametrize("method", ["rbcg", "rbi"])
def test_nonfinite_rhs(orc, rbs, method):
    """NaN / Inf in a query's right-hand side: NONFINITE for that query only (AMB-11)."""
    import torch
    g, tr, res = _small2d(orc)
    s = rbs.Solver(2, 15, (2, 2)).load_basis(res["W"], res["ANq"], res["fn"])
    rhs = np.ones((4, g.N))
    rhs[1, 7] = np.nan
    rhs[2, 100] = np.inf
    kw = dict(method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI,
              max_iter=20000 if method == "rbcg" else 500000)
    out = s.solve_batch(tr[:4], rhs=torch.tensor(rhs, device="cuda"), **kw)
    solve = g.rbcg if method == "rbcg" else g.rbi
    for b in range(4):
        ref = solve(res["W"], res["ANq"], res["fn"], tr[b], b=rhs[b], max_iter=kw["max_iter"])
        assert out["status"][b] == ref["status"], (b, out["status"][b], ref["status"])
    assert out["status"][1] == out["status"][2] == "NONFINITE" and out["its"][1] == out["its"][2] == 0
    for b in (0, 3):
        ref = solve(res["W"], res["ANq"], res["fn"], tr[b], b=rhs[b], max_iter=kw["max_iter"])
        assert abs(int(out["its"][b]) - ref["its"]) <= 1
        x = out["X"][b].cpu().numpy()
        assert np.linalg.norm(x - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])


@pytest.mark.parametrize("dim,m", [(2, 1), (2, 2), (2, 3), (2, 7), (3, 1), (3, 2), (3, 3), (3, 7)])
@pytest.mark.parametrize("method", ["rbcg", "rbi"])
def test_tiny_grids(orc, rbs, dim, m, method):
    """The smallest grids (m = 1, 2, 3, 7): one-node grids, strips and row
    segments shorter than every tile; B = 1 and B = 3."""
    g = orc.Grid(dim, m, (2,) * dim)
    tr = 0.1 * 100 ** np.random.default_rng(m).random((10, g.Q))
    res = g.greedy(tr, min(3, g.N))
    s = rbs.Solver(dim, m, (2,) * dim).load_basis(res["W"], res["ANq"], res["fn"])
    mi = 20000 if method == "rbcg" else 500000
    kw = dict(method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI, max_iter=mi, record_history=1)
    for mus in (tr[3:4], tr[4:7]):
        out = s.solve_batch(mus, **kw)
        compare(out, g, res["W"], res["ANq"], res["fn"], mus, method, max_iter=mi)


def test_single_query_batches_match_the_batch(orc, rbs):
    """B = 1 solves of every c1 query against the oracle (the row-march kernels at their
    narrowest batch) and against the same queries solved as one batch of 8."""
    c = CONFIGS["c1"]
    g = orc.Grid(c.dim, c.m, c.blocks)
    from synth import train_set
    res = g.greedy(train_set(c), c.n)
    s = rbs.Solver(c.dim, c.m, c.blocks).load_basis(res["W"], res["ANq"], res["fn"])
    mus = query_set(c)
    full = s.solve_batch(mus, record_history=1)
    for b in range(len(mus)):
        one = s.solve_batch(mus[b:b + 1], record_history=1)
        compare(one, g, res["W"], res["ANq"], res["fn"], mus[b:b + 1], "rbcg")
        assert one["status"][0] == full["status"][b] and abs(int(one["its"][0]) - int(full["its"][b])) <= 1
        x1, xb = one["X"][0].cpu().numpy(), full["X"][b].cpu().numpy()
        assert np.linalg.norm(x1 - xb) <= 1e-11 * np.linalg.norm(xb)


def test_batch_composition_invariance(orc, rbs):
    """a query's iterates do not depend on its position in the
    batch or on the other queries -- bitwise for batches of the same padded width (every
    per-query sum runs over the same nodes in the same order), to rounding across widths
    (the kernels' thread-to-node maps, hence the partial-sum order, depend on the width)."""
    g, res = oracle_basis(orc, 2, 63, (3, 3), 12, 40, 2)
    s = rbs.Solver(2, 63, (3, 3)).load_basis(res["W"], res["ANq"], res["fn"])
    rng = np.random.default_rng(77)
    pool = 0.1 * 100 ** rng.random((40, 9))
    base = s.solve_batch(pool[:24], record_history=1)              # width 32
    perm = rng.permutation(24)
    pb = s.solve_batch(pool[perm], record_history=1)               # same width, other positions
    mixed = s.solve_batch(np.vstack([pool[30:40], pool[:20]]), record_history=1)   # width 32, new companions
    X0, Xp, Xm = base["X"].cpu().numpy(), pb["X"].cpu().numpy(), mixed["X"].cpu().numpy()
    for i in range(24):
        j = int(np.where(perm == i)[0][0])
        assert np.array_equal(X0[i], Xp[j]) and np.array_equal(base["history"][i], pb["history"][j])
        if i < 20:
            assert np.array_equal(X0[i], Xm[10 + i]) and base["its"][i] == mixed["its"][10 + i]
    for w in (1, 5, 16):                                           # other widths: to rounding
        o = s.solve_batch(pool[:w], record_history=1)
        Xo = o["X"].cpu().numpy()
        for i in range(w):
            assert abs(int(o["its"][i]) - int(base["its"][i])) <= 1
            assert np.linalg.norm(Xo[i] - X0[i]) <= 1e-11 * np.linalg.norm(X0[i])
