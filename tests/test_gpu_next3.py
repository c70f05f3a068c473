"""NEXT(3) variants on the GPU against the oracle: the symmetric
two-level RBI preconditioner (adjoint pre-smoothing + coarse correction + post-smoothing,
RBS_PRECOND_SYM) and the Polak-Ribiere / flexible beta (RBS_BETA_PR), 2D and 3D, with the
red-black smoothers and damped Jacobi.  Criteria as tests/test_gpu_parity.py."""
import numpy as np
import pytest

from test_gpu_parity import compare, oracle_basis, rbs  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dim,m,blocks,n,B", [(2, 63, (2, 2), 16, 8), (2, 40, (3, 3), 10, 13),
                                              (3, 13, (2, 2, 2), 8, 6)])
@pytest.mark.parametrize("precond,beta", [(1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("smoother", [0, 1, 2])
def test_precond_and_beta_variants(orc, rbs, dim, m, blocks, n, B, precond, beta, smoother):
    g, res = oracle_basis(orc, dim, m, blocks, n, max(30, n + 20), 3)
    s = rbs.Solver(dim, m, blocks).load_basis(res["W"], res["ANq"], res["fn"])
    mus = 0.1 * 100 ** np.random.default_rng(200 + m).random((B, g.Q))
    kw = dict(smoother=smoother, omega=0.8 if smoother == 2 else 1.0)
    out = s.solve_batch(mus, record_history=1, precond=precond, beta_rule=beta, **kw)
    assert all(st == "CONVERGED" for st in out["status"]), out["status"]
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbcg", precond=precond, beta_rule=beta, **kw)


def test_symmetric_precond_fixed_iterations(orc, rbs):
    """tol = 0, K fixed: x_K parity of the symmetric two-level preconditioner (drift-free)."""
    g, res = oracle_basis(orc, 2, 45, (3, 3), 10, 30, 3)
    s = rbs.Solver(2, 45, (3, 3)).load_basis(res["W"], res["ANq"], res["fn"])
    mus = 0.1 * 100 ** np.random.default_rng(4).random((8, 9))
    out = s.solve_batch(mus, tol=0.0, max_iter=25, record_history=1, precond=1, beta_rule=1)
    assert all(st == "MAXIT" for st in out["status"]) and np.all(out["its"] == 25)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbcg", tol=0.0, max_iter=25, precond=1, beta_rule=1)


def test_variant_errors(rbs):
    s = rbs.Solver(2, 20, (2, 2))
    s.load_basis(np.linalg.qr(np.random.default_rng(0).standard_normal((400, 3)))[0])
    with pytest.raises(rbs.RbsError, match="E_ARG"):
        s.solve_batch(np.ones((2, 4)), method=rbs.RBS_RBI, precond=1)
    with pytest.raises(rbs.RbsError, match="E_ARG"):
        s.solve_batch(np.ones((2, 4)), beta_rule=7)
