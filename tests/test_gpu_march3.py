"""k_smooth3 (march3.cuh, K3 with register windows) against k_smooth2 and the oracle.

k_smooth3 evaluates every node with k_smooth2's formulas in the same order (same
DMMA accumulation chain, same direct-form Gauss-Seidel value), so the smoothed
vectors agree BITWISE (RBI; RBCG to rounding, its y^T r sums are split differently); parity with the oracle then follows from k_smooth2's (and is
checked directly here too).  RBS_DISABLE_V2 bit 2048 (read at context creation)
turns k_smooth3 off.
"""
import os

import numpy as np
import pytest

from test_gpu_parity import compare, oracle_basis, rbs  # noqa: F401  (fixture)
from synth import CONFIGS, query_set, train_set

pytestmark = pytest.mark.gpu


def _pair(rbs, dim, m, blocks, W, ANq, fn):
    a = rbs.Solver(dim, m, blocks).load_basis(W, ANq, fn)
    old = os.environ.get("RBS_DISABLE_V2")
    os.environ["RBS_DISABLE_V2"] = "2048"
    try:
        b = rbs.Solver(dim, m, blocks).load_basis(W, ANq, fn)
    finally:
        if old is None:
            del os.environ["RBS_DISABLE_V2"]
        else:
            os.environ["RBS_DISABLE_V2"] = old
    return a, b


def _same(x, y, bitwise=True):
    """bitwise: RBI (K3 has no reduction); RBCG: the y^T r partial sums of the two
    kernels are accumulated in a different order (another thread / slot split), so
    beta differs in the last bits and the iterates agree to rounding only."""
    assert list(x["status"]) == list(y["status"])
    assert np.array_equal(x["its"], y["its"])
    xa, ya = x["X"].cpu().numpy(), y["X"].cpu().numpy()
    if bitwise:
        assert np.array_equal(xa, ya)
    else:
        assert np.linalg.norm(xa - ya) <= 1e-12 * np.linalg.norm(ya)
    if "history" in x:
        for hx, hy in zip(x["history"], y["history"]):
            if bitwise:
                assert np.array_equal(hx, hy)
            else:
                assert np.all(np.abs(hx - hy) <= 1e-8 * np.abs(hy) + 1e-15)


@pytest.mark.parametrize("m,blocks,n,B", [(63, (3, 3), 40, 32), (100, (2, 3), 16, 32), (37, (3, 3), 60, 32),
                                          (81, (3, 3), 8, 20)])
@pytest.mark.parametrize("method,smoother", [("rbcg", 0), ("rbcg", 1), ("rbi", 0), ("rbi", 1)])
def test_smooth3_bitwise_equals_smooth2_and_oracle(orc, rbs, m, blocks, n, B, method, smoother):
    g, res = oracle_basis(orc, 2, m, blocks, n, max(30, n + 20), 2)
    s3, s2 = _pair(rbs, 2, m, blocks, res["W"], res["ANq"], res["fn"])
    mus = 0.1 * 100 ** np.random.default_rng(300 + m).random((B, g.Q))
    mi = 20000 if method == "rbcg" else 500000
    kw = dict(method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI, max_iter=mi, record_history=1,
              smoother=smoother)
    x3 = s3.solve_batch(mus, **kw)
    x2 = s2.solve_batch(mus, **kw)
    _same(x3, x2, bitwise=method == "rbi")
    idx = [0, B // 2, B - 1]
    compare(dict(x3, X=x3["X"][idx], status=[x3["status"][i] for i in idx], its=x3["its"][idx],
                 a_n=x3["a_n"][idx], history=[x3["history"][i] for i in idx]),
            g, res["W"], res["ANq"], res["fn"], mus[idx], method, max_iter=mi, smoother=smoother)


def test_smooth3_rbi_rhs_override(orc, rbs):
    """RBI with per-query right-hand sides: x_old accumulation and rhs rows together."""
    import torch
    g, res = oracle_basis(orc, 2, 63, (3, 3), 12, 40, 2)
    s3, s2 = _pair(rbs, 2, 63, (3, 3), res["W"], res["ANq"], res["fn"])
    rng = np.random.default_rng(5)
    mus = 0.1 * 100 ** rng.random((32, 9))
    rhs = rng.standard_normal((32, g.N))
    rt = torch.tensor(rhs, device="cuda")
    kw = dict(method=rbs.RBS_RBI, tol=0.0, max_iter=60, record_history=1)
    x3 = s3.solve_batch(mus, rhs=rt, **kw)
    x2 = s2.solve_batch(mus, rhs=rt, **kw)
    _same(x3, x2)
    for b in (0, 31):
        ref = g.rbi(res["W"], res["ANq"], res["fn"], mus[b], b=rhs[b], tol=0.0, max_iter=60)
        x = x3["X"][b].cpu().numpy()
        assert np.linalg.norm(x - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])


def test_smooth3_c2_full_size_bitwise(orc, rbs):
    """The bench configuration (c2: 511^2, n = 40, B = 32): k_smooth3 and k_smooth2 give the
    same iterates bit for bit over a fixed 40-iteration RBCG run."""
    c = CONFIGS["c2"]
    W, ANq, fn = orc.interpolated_basis(c.dim, c.m, c.blocks, train_set(c), c.n, 63)
    s3, s2 = _pair(rbs, c.dim, c.m, c.blocks, W, ANq, fn)
    mus = query_set(c)[:c.B]
    kw = dict(tol=0.0, max_iter=40, record_history=1)
    _same(s3.solve_batch(mus, **kw), s2.solve_batch(mus, **kw), bitwise=False)
    kw = dict(method=rbs.RBS_RBI, tol=0.0, max_iter=40, record_history=1)
    _same(s3.solve_batch(mus, **kw), s2.solve_batch(mus, **kw))
