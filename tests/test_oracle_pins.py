"""Pins of the CPU oracle against things other than itself.

Every test here is `not gpu`.  Sources: closed forms (Laplacian eigenpairs),
an independent P1-FEM assembly (PAPER.md:319 discretisation), textbook SGS-PCG
(scipy), LAPACK, the paper's Lemmas 1-3, Galerkin
optimality, and SPEC.md worked examples (tests/golden/spec_examples.json).
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import refs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
RNG = np.random.default_rng(12345)


def rand_mu(Q, lo=0.1, hi=10.0, rng=RNG):
    return lo * (hi / lo) ** rng.random(Q)


# --------------------------------------------------------------------------- operator
@pytest.mark.parametrize("dim,m,blocks", [(2, 7, (2, 2)), (2, 12, (3, 3)), (3, 5, (2, 2, 2)),
                                          (3, 6, (2, 3, 2))])
def test_operator_equals_cellwise_assembly(orc, dim, m, blocks):
    g = orc.Grid(dim, m, blocks)
    mu = rand_mu(g.Q)
    A = g.dense_A(mu)
    R = refs.cellwise_fd(dim, m, blocks, mu).toarray()
    assert np.abs(A - R).max() <= 1e-13 * np.abs(R).max()
    assert np.array_equal(A, A.T)  # bitwise symmetric


@pytest.mark.parametrize("m,blocks", [(7, (2, 2)), (11, (3, 3)), (8, (2, 2))])
@pytest.mark.parametrize("diag", ["main", "anti"])
def test_operator_equals_p1_fem_2d(orc, m, blocks, diag):
    """AMB-1: the cell-averaged 5-point system is the P1-FEM system."""
    g = orc.Grid(2, m, blocks)
    mu = rand_mu(g.Q)
    K = refs.fem_p1_2d(m, blocks, mu, diag).toarray()
    A = g.dense_A(mu)
    h2 = 1.0 / (m + 1) ** 2
    assert np.abs(h2 * A - K).max() <= 1e-13 * np.abs(K).max()
    # FEM load of f = 1 is h^2 per node: A x = 1 <=> K x = load
    assert np.allclose(refs.fem_load_2d(m), h2 * np.ones(m * m), rtol=0, atol=1e-18)


@pytest.mark.parametrize("dim,m,ks", [(2, 15, (1, 1)), (2, 15, (3, 7)), (2, 16, (16, 2)),
                                      (3, 7, (1, 2, 3)), (3, 8, (8, 1, 5))])
def test_constant_theta_is_scaled_laplacian(orc, dim, m, ks):
    """theta == c: A v = c lambda v for the sine eigenvectors (closed form)."""
    blocks = (2,) * dim
    g = orc.Grid(dim, m, blocks)
    c = 2.75
    lam, v = refs.laplacian_eig(dim, m, ks)
    Av = g.apply_A(np.full(g.Q, c), v)
    assert np.abs(Av - c * lam * v).max() <= 1e-12 * c * lam


def test_affine_linearity(orc):
    """A(theta) = sum_q theta_q A(e_q)."""
    g = orc.Grid(3, 6, (2, 2, 2))
    mu = rand_mu(g.Q)
    x = RNG.standard_normal(g.N)
    tot = np.zeros(g.N)
    for q in range(g.Q):
        e = np.zeros(g.Q); e[q] = 1.0
        tot += mu[q] * g.apply_A(e, x)
    ref = g.apply_A(mu, x)
    assert np.abs(tot - ref).max() <= 1e-13 * np.abs(ref).max() * g.Q


def test_Aq_psd_and_A_spd(orc):
    g = orc.Grid(2, 9, (3, 3))
    for q in range(g.Q):
        e = np.zeros(g.Q); e[q] = 1.0
        assert np.linalg.eigvalsh(g.dense_A(e)).min() > -1e-10
    L, piv = orc.cholesky(g.dense_A(rand_mu(g.Q)))
    assert piv == -1


# --------------------------------------------------------------------------- smoother
@pytest.mark.parametrize("dim,m,blocks", [(2, 6, (2, 2)), (2, 7, (3, 3)), (3, 4, (2, 2, 2))])
def test_rbgs_is_textbook_gs_in_red_black_order(orc, dim, m, blocks):
    g = orc.Grid(dim, m, blocks)
    mu = rand_mu(g.Q)
    A = refs.cellwise_fd(dim, m, blocks, mu).toarray()
    b = RNG.standard_normal(g.N)
    y0 = RNG.standard_normal(g.N)
    order = refs.red_black_order(dim, m)
    # textbook forward GS in red-then-black order
    y = y0.copy()
    for i in order:
        y[i] = (b[i] - A[i] @ y + A[i, i] * y[i]) / A[i, i]
    red = g.gs_halfsweep(mu, b, y0, 0)
    got = g.gs_halfsweep(mu, b, red, 1)
    assert np.abs(got - y).max() <= 1e-13 * np.abs(y).max()
    assert np.array_equal(g.smooth(mu, b, y0, orc.FWD_RBGS, 1), got)
    # (1,1[,1]) colour convention: first interior node red in 2D, black in 3D
    par = dim % 2
    assert (red[0] != y0[0]) == (par == 0)


@pytest.mark.parametrize("dim,m,blocks,omega,sweeps", [(2, 7, (3, 3), 1.0, 1), (2, 6, (2, 2), 0.8, 2),
                                                       (3, 4, (2, 2, 2), 2.0 / 3.0, 3)])
def test_jacobi_is_textbook_damped_jacobi(orc, dim, m, blocks, omega, sweeps):
    """S = Jacobi ("the smoother (Jacobi or Gauss-Seidel)"): each sweep is
    y <- y + omega D^-1 (b - A y) on the independently assembled matrix (tests/refs.py)."""
    g = orc.Grid(dim, m, blocks)
    mu = rand_mu(g.Q)
    A = refs.cellwise_fd(dim, m, blocks, mu).toarray()
    b = RNG.standard_normal(g.N)
    y = RNG.standard_normal(g.N)
    got = g.smooth(mu, b, y, orc.JACOBI, sweeps, omega)
    d = np.diag(A)
    for _ in range(sweeps):
        y = y + omega * (b - A @ y) / d
    assert np.abs(got - y).max() <= 1e-12 * np.abs(y).max()


def test_jacobi_contracts_on_the_laplacian(orc):
    """undamped Jacobi does not increase ||x - x*||_inf on the constant-
    coefficient Laplacian (||D^-1 (L + U)||_inf = 1) and reduces it over sweeps; x* is fixed."""
    g = orc.Grid(2, 9, (2, 2))
    mu = np.ones(g.Q)
    A = refs.cellwise_fd(2, 9, (2, 2), mu).toarray()
    b = RNG.standard_normal(g.N)
    xs = np.linalg.solve(A, b)
    assert np.abs(g.smooth(mu, b, xs, orc.JACOBI, 1, 1.0) - xs).max() <= 1e-13 * np.abs(xs).max()
    y = RNG.standard_normal(g.N)
    e0 = np.abs(y - xs).max()
    for _ in range(4):
        y2 = g.smooth(mu, b, y, orc.JACOBI, 1, 1.0)
        assert np.abs(y2 - xs).max() <= np.abs(y - xs).max() * (1 + 1e-14)   # ||J||_inf = 1
        y = y2
    assert np.abs(y - xs).max() < e0


def test_symmetric_rbgs_is_rbr_bitwise(orc):
    """R,B,B,R == R,B,R bitwise (the repeated black half-sweep is a no-op, AMB-6)."""
    g = orc.Grid(2, 13, (3, 3))
    mu = rand_mu(g.Q)
    b = RNG.standard_normal(g.N)
    y0 = RNG.standard_normal(g.N)
    y = g.gs_halfsweep(mu, b, y0, 0)
    y = g.gs_halfsweep(mu, b, y, 1)
    y = g.gs_halfsweep(mu, b, y, 0)
    assert np.array_equal(g.smooth(mu, b, y0, orc.SYM_RBGS, 1), y)


def test_smoother_fixed_point_and_energy(orc):
    g = orc.Grid(2, 11, (2, 2))
    mu = rand_mu(g.Q)
    A = refs.cellwise_fd(2, 11, (2, 2), mu).toarray()
    b = RNG.standard_normal(g.N)
    xs = np.linalg.solve(A, b)
    for kind in (orc.SYM_RBGS, orc.FWD_RBGS):
        z = g.smooth(mu, b, xs, kind, 1)
        assert np.abs(z - xs).max() <= 1e-13 * np.abs(xs).max()
    y = RNG.standard_normal(g.N)
    en = lambda v: np.sqrt((v - xs) @ A @ (v - xs))
    for _ in range(5):
        y2 = g.smooth(mu, b, y, orc.SYM_RBGS, 1)
        assert en(y2) <= en(y) * (1 + 1e-14)
        y = y2


# --------------------------------------------------------------------------- dense
def test_spec_cholesky_examples(orc):
    for ex in GOLD["cholesky"]:
        L, piv = orc.cholesky(np.array(ex["M"]))
        assert piv == -1 and np.allclose(L, ex["L"], atol=1e-15), ex["cite"]
    for ex in GOLD["cholesky_fail"]:
        _, piv = orc.cholesky(np.array(ex["M"]))
        assert piv == ex["pivot"], ex["cite"]
    for ex in GOLD["chol_solve"]:
        L, _ = orc.cholesky(np.array(ex["M"]))
        assert np.allclose(orc.chol_solve(L, np.array(ex["b"])), ex["x"], atol=1e-15), ex["cite"]
    for ex in GOLD["dot"]:
        assert orc.dot(np.array(ex["x"]), np.array(ex["y"])) == ex["value"]


@pytest.mark.parametrize("n", [1, 5, 17, 40, 64])
def test_cholesky_vs_lapack(orc, n):
    X = RNG.standard_normal((n, n))
    M = X @ X.T + n * np.eye(n)
    L, piv = orc.cholesky(M)
    assert piv == -1
    assert np.abs(L - np.linalg.cholesky(M)).max() <= 1e-12 * np.abs(L).max()
    b = RNG.standard_normal(n)
    assert np.abs(orc.chol_solve(L, b) - np.linalg.solve(M, b)).max() <= 1e-10 * np.abs(
        np.linalg.solve(M, b)).max()
    # leading principal block identity (AMB-19)
    k = max(1, n // 2)
    Lk, _ = orc.cholesky(M[:k, :k])
    assert np.array_equal(Lk, L[:k, :k])


def test_dot_is_compensated(orc):
    x = np.array([1e16, 1.0, -1e16, 1.0])
    assert orc.dot(x, np.ones(4)) == 2.0


def test_spec_mgs_examples(orc):
    for ex in GOLD["mgs"]:
        W = np.array(ex["W"]).T
        Wn, rej = orc.mgs_append(W, np.array(ex["v"]))
        if ex.get("rejected"):
            assert rej, ex["cite"]
        else:
            assert not rej and np.allclose(Wn[:, -1], ex["new"], atol=1e-15), ex["cite"]
    W = None
    for _ in range(12):
        W, rej = orc.mgs_append(W, RNG.standard_normal(300))
        assert not rej
    assert np.abs(W.T @ W - np.eye(12)).max() < 1e-14
    _, rej = orc.mgs_append(W, W @ RNG.standard_normal(12))  # dependent vector
    assert rej


# --------------------------------------------------------------------------- basis / solvers
@pytest.fixture(scope="module")
def small2d(orc):
    g = orc.Grid(2, 15, (2, 2))
    tr = 0.1 * 100 ** np.random.default_rng(7).random((40, 4))
    res = g.greedy(tr, 8)
    return g, tr, res


def test_offline_online_consistency(orc, small2d):
    """sum_q theta_q A_{n,q} = W^T A(theta) W and f_n = W^T f."""
    g, _, res = small2d
    W, ANq, fn = res["W"], res["ANq"], res["fn"]
    assert np.abs(W.T @ W - np.eye(res["n"])).max() < 1e-12
    ANq2, fn2 = g.offline_blocks(W)
    assert np.abs(ANq2 - ANq).max() <= 1e-12 * np.abs(ANq).max()  # incremental == recompute
    for q in range(g.Q):
        assert np.array_equal(ANq[q], ANq[q].T)
    for _ in range(20):
        mu = rand_mu(g.Q)
        A = refs.cellwise_fd(2, g.m, g.blocks, mu).toarray()
        An = np.einsum("q,qij->ij", mu, ANq)
        ref = W.T @ A @ W
        assert np.abs(An - ref).max() <= 1e-12 * np.abs(ref).max()
        assert np.linalg.eigvalsh(An).min() > 0
    assert np.abs(fn - W.T @ np.ones(g.N)).max() <= 1e-12 * np.abs(fn).max()


def test_lemma1_rbi_and_rbcg_one_iteration(orc, small2d):
    """x in span(W) => RBI and RBCG converge in one iteration."""
    g, _, res = small2d
    W, ANq, fn = res["W"], res["ANq"], res["fn"]
    mu = rand_mu(g.Q)
    c = RNG.standard_normal(res["n"])
    b = g.apply_A(mu, W @ c)
    for solve in (g.rbi, g.rbcg):
        out = solve(W, ANq, fn, mu, b=b)
        assert out["status"] == "CONVERGED" and out["its"] == 1
        assert np.linalg.norm(out["x"] - W @ c) <= 1e-10 * np.linalg.norm(W @ c)
        assert np.abs(out["a_n"] - c).max() <= 1e-10 * np.abs(c).max()


def test_lemma2_stagnation_without_smoother(orc, small2d):
    """sweeps = 0 => x_k = x_hat for all k >= 1, MAXIT."""
    g, _, res = small2d
    W, ANq, fn = res["W"], res["ANq"], res["fn"]
    mu = rand_mu(g.Q)
    xhat = W @ orc.rb_solve(ANq, fn, mu)[0]
    for k in (1, 2, 5):
        out = g.rbi(W, ANq, fn, mu, sweeps=0, max_iter=k)
        assert out["status"] == "MAXIT"
        assert np.linalg.norm(out["x"] - xhat) <= 1e-12 * np.linalg.norm(xhat)
    # RBCG with nu = 0: W^T r_1 = 0 so the second preconditioner gives rho' ~ 0
    out = g.rbcg(W, ANq, fn, mu, sweeps=0)
    assert out["status"] == "PRECOND" and out["its"] == 1


def test_lemma3_galerkin_orthogonality(orc, small2d):
    """W e_n is the RB approximation of the error: after one
    RBI step without smoothing, W^T (f - A x) = 0."""
    g, _, res = small2d
    W, ANq, fn = res["W"], res["ANq"], res["fn"]
    mu = rand_mu(g.Q)
    b = RNG.standard_normal(g.N)
    out = g.rbi(W, ANq, fn, mu, b=b, sweeps=0, max_iter=1)
    r = b - g.apply_A(mu, out["x"])
    assert np.linalg.norm(W.T @ r) <= 1e-12 * np.linalg.norm(W.T @ b)


@pytest.mark.parametrize("dim,m,blocks", [(2, 15, (2, 2)), (3, 7, (2, 2, 2))])
def test_solvers_reach_direct_solution(orc, dim, m, blocks):
    g = orc.Grid(dim, m, blocks)
    rng = np.random.default_rng(3)
    tr = 0.1 * 100 ** rng.random((30, g.Q))
    res = g.greedy(tr, 6)
    for mu in 0.1 * 100 ** rng.random((3, g.Q)):
        A = refs.cellwise_fd(dim, m, blocks, mu).tocsc()
        xs = spla.spsolve(A, np.ones(g.N))
        for solve in (g.rbcg, g.rbi):
            out = solve(res["W"], res["ANq"], res["fn"], mu)
            assert out["status"] == "CONVERGED"
            assert out["true_relres"] < 1e-10
            assert np.linalg.norm(out["x"] - xs) <= 1e-8 * np.linalg.norm(xs)
            assert out["hist"][-1] < 1e-10 and len(out["hist"]) == out["its"] + 1


def test_constant_theta_solution_matches_closed_form(orc):
    """theta == c: x* = sum_k (<v_k,1>/|v_k|^2)/(c lambda_k) v_k (DST, closed form)."""
    m, c = 15, 3.5
    g = orc.Grid(2, m, (2, 2))
    xs = np.zeros(g.N)
    for k1 in range(1, m + 1):
        for k2 in range(1, m + 1):
            lam, v = refs.laplacian_eig(2, m, (k1, k2))
            xs += (v @ np.ones(g.N)) / (v @ v) / (c * lam) * v
    out = g.rbcg(None, None, None, np.full(4, c))
    assert out["status"] == "CONVERGED"
    assert np.linalg.norm(out["x"] - xs) <= 1e-9 * np.linalg.norm(xs)


@pytest.mark.parametrize("dim,m,blocks", [(2, 20, (3, 3)), (3, 7, (2, 2, 2))])
def test_empty_basis_rbcg_is_ssor_pcg(orc, dim, m, blocks):
    """n = 0: RBCG = CG preconditioned by symmetric RB-GS (textbook SGS-PCG)."""
    g = orc.Grid(dim, m, blocks)
    mu = rand_mu(g.Q, rng=np.random.default_rng(11))
    A = refs.cellwise_fd(dim, m, blocks, mu).tocsr()
    order = refs.red_black_order(dim, m)
    M = spla.LinearOperator(A.shape, matvec=lambda r: refs.sgs_rb_apply(A, order, r))
    count = [0]
    b = np.ones(g.N)
    spla.cg(A, b, M=M, rtol=1e-10, atol=0.0, maxiter=5000,
            callback=lambda xk: count.__setitem__(0, count[0] + 1))
    out = g.rbcg(None, None, None, mu)
    assert out["status"] == "CONVERGED"
    assert abs(out["its"] - count[0]) <= 1


def test_rbcg_fewer_iterations_than_cg(orc):
    """context: RBCG << CG on a family with fast n-width decay."""
    g = orc.Grid(2, 31, (2, 2))
    rng = np.random.default_rng(5)
    res = g.greedy(0.1 * 100 ** rng.random((40, 4)), 8)
    mu = 0.1 * 100 ** rng.random(4)
    assert g.rbcg(res["W"], res["ANq"], res["fn"], mu)["its"] * 3 < g.cg(mu)["its"]


# --------------------------------------------------------------------------- greedy
def test_greedy_first_vector_is_normalised_snapshot(orc):
    g = orc.Grid(2, 12, (2, 2))
    tr = 0.1 * 100 ** np.random.default_rng(9).random((10, 4))
    res = g.greedy(tr, 1)
    xs = spla.spsolve(refs.cellwise_fd(2, 12, (2, 2), tr[0]).tocsc(), np.ones(g.N))
    w = xs / np.linalg.norm(xs)
    assert res["selected"][0] == 0
    assert np.linalg.norm(res["W"][:, 0] - w) <= 1e-10


def test_greedy_energy_error_monotone(orc):
    """AMB-16: max over Xi_train of ||x - W_N a_N||_A is nonincreasing in N."""
    g = orc.Grid(2, 13, (3, 3))
    rng = np.random.default_rng(21)
    tr = 0.1 * 100 ** rng.random((25, 9))
    res = g.greedy(tr, 8)
    W, ANq, fn = res["W"], res["ANq"], res["fn"]
    truth = []
    for mu in tr:
        A = refs.cellwise_fd(2, 13, (3, 3), mu).tocsc()
        truth.append((A, spla.spsolve(A, np.ones(g.N))))
    prev = np.full(len(tr), np.inf)
    for N in range(1, res["n"] + 1):
        errs = []
        for t, mu in enumerate(tr):
            A, xs = truth[t]
            a, piv = orc.rb_solve(ANq[:, :N, :N].copy(), fn[:N].copy(), mu)
            d = xs - W[:, :N] @ a
            e = np.sqrt(max(d @ (A @ d), 0.0))
            floor = 1e-13 * np.sqrt(xs @ (A @ xs))
            assert e <= prev[t] * (1 + 1e-9) + floor
            errs.append(e)
        prev = np.array(errs)


def test_greedy_rejects_dependent_snapshot(orc):
    """2 mu = scaled copies => x(2mu) = x(mu)/2 is dependent and is rejected."""
    g = orc.Grid(2, 10, (2, 2))
    mu = np.array([1.0, 2.0, 0.5, 3.0])
    res = g.greedy(np.vstack([mu, 2 * mu]), 2)
    assert res["n"] == 1 and res["n_rejected"] == 1


def test_greedy_deterministic_and_plain_equals_adaptive(orc):
    g = orc.Grid(2, 15, (2, 2))
    tr = 0.1 * 100 ** np.random.default_rng(4).random((30, 4))
    r1 = g.greedy(tr, 6)
    r2 = g.greedy(tr, 6)
    assert np.array_equal(r1["W"], r2["W"]) and np.array_equal(r1["selected"], r2["selected"])
    r3 = g.greedy(tr, 6, adaptive=False)
    assert np.array_equal(r1["selected"], r3["selected"])
    s = np.linalg.svd(r1["W"].T @ r3["W"], compute_uv=False)
    assert s.min() > 1 - 1e-10  # principal angles ~ 0


def test_multifidelity_basis(orc):
    """samples from a coarse greedy, snapshots on the fine grid."""
    tr = 0.1 * 100 ** np.random.default_rng(8).random((30, 4))
    coarse = orc.Grid(2, 15, (2, 2)).greedy(tr, 5)
    fine = orc.Grid(2, 31, (2, 2))
    mf = fine.basis_from_samples(tr[coarse["selected"]])
    assert mf["n"] == 5
    assert np.abs(mf["W"].T @ mf["W"] - np.eye(5)).max() < 1e-12
    out = fine.rbcg(mf["W"], mf["ANq"], mf["fn"], tr[3])
    assert out["status"] == "CONVERGED"


# --------------------------------------------------------------------------- adaptive n (NEXT(2))
def test_adapt_n_rule_spec_examples(orc):
    """The gamma-rule of PAPER.md:287 on SPEC's worked examples (golden, cited)."""
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
    for ex in gold["adapt_n"]:
        assert orc.adapt_n(ex["ratio"], 1.0, ex["gamma"], ex["na"], ex["n_max"]) == ex["out"], ex["cite"]
    assert orc.adapt_n(2.0, 1.0, 0.0, 3, 8) == 3          # gamma = 0: rule off


@pytest.mark.parametrize("k", [1, 3, 5])
def test_active_dimension_is_the_truncated_basis(orc, small2d, k):
    """Using the leading k columns (n_active = k) is the RB method with W_k: the
    Cholesky factor of a leading principal block is the leading block of the full
    factor, so the solves equal those of the truncated basis (W[:, :k], the k x k
    leading blocks of A_{n,q}, f_n[:k]) -- bitwise, same operation order."""
    g, _, res = small2d
    W, ANq, fn = res["W"], res["ANq"], res["fn"]
    Wk, Ak, fk = np.asfortranarray(W[:, :k]), np.ascontiguousarray(ANq[:, :k, :k]), fn[:k].copy()
    mu = rand_mu(g.Q)
    for solve, kw in ((g.rbcg, {}), (g.rbi, {})):
        a = solve(W, ANq, fn, mu, n_active=k, **kw)
        b = solve(Wk, Ak, fk, mu, **kw)
        assert a["status"] == b["status"] and a["its"] == b["its"]
        assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["hist"], b["hist"])
        assert np.array_equal(a["a_n"][:k], b["a_n"]) and not np.any(a["a_n"][k:])
    c = g.rbcg(W, ANq, fn, mu, n_active=k, gamma=0.0)
    assert np.array_equal(c["x"], g.rbcg(Wk, Ak, fk, mu)["x"]) and np.all(c["active_n"] == k)


def test_adaptive_n_grows_by_the_rule_and_converges(orc, small2d):
    """gamma = 10 from n_active = 1: the active dimension is nondecreasing, grows by at
    most one per iteration exactly when the residual ratio is below gamma (checked
    against the returned history), stays <= n, and the iterate reaches the direct
    solution."""
    g, _, res = small2d
    W, ANq, fn = res["W"], res["ANq"], res["fn"]
    mu = rand_mu(g.Q)
    out = g.rbcg(W, ANq, fn, mu, n_active=1, gamma=10.0)
    act, h = out["active_n"], out["hist"]
    assert out["status"] == "CONVERGED" and act[0] == 1
    assert np.all(np.diff(act) >= 0) and np.all(np.diff(act) <= 1) and act.max() <= res["n"]
    for k in range(out["its"] - 1):
        grow = h[k] / h[k + 1] < 10.0 and act[k] < res["n"]
        assert act[k + 1] == act[k] + (1 if grow else 0), k
    A = refs.cellwise_fd(2, g.m, g.blocks, mu).toarray()
    xs = np.linalg.solve(A, np.ones(g.N))
    assert np.linalg.norm(out["x"] - xs) <= 1e-8 * np.linalg.norm(xs)


# --------------------------------------------------------------------------- greedy Steps 5-6 (recomputed)
def _recompute_selection(dim, m, blocks, tr, W, selected, n_out, rhs=None):
    """Steps 5-6 of algorithm0/algorithm3 recomputed from
    their definition with independent pieces: for N = 1..n-1, A_N(mu_t) = W_N^T A(mu_t)
    W_N with A from the cell-wise assembly (refs.cellwise_fd), f_N = W_N^T f(mu_t),
    a_N(mu_t) by numpy.linalg.solve, indicator = sum_j |a_N,j| (the L1 norm of
    PAPER.md:87); mu_{N+1} = argmax over the parameters not selected yet, lowest index
    on ties (AMB-13).  Returns, per step, (expected index, top-2 gap, max indicator)."""
    out = []
    As = [refs.cellwise_fd(dim, m, blocks, mu).tocsr() for mu in tr]
    for N in range(1, n_out):
        WN = W[:, :N]
        ind = np.empty(len(tr))
        for t, A in enumerate(As):
            f = np.ones(W.shape[0]) if rhs is None else rhs(t)
            ind[t] = np.abs(np.linalg.solve(WN.T @ (A @ WN), WN.T @ f)).sum()
        ind[list(selected[:N])] = -np.inf
        best = int(np.argmax(ind))          # numpy: first (lowest) index of the maximum
        srt = np.sort(ind)[::-1]
        out.append((best, (srt[0] - srt[1]) / srt[0], srt[0]))
    return out


@pytest.mark.parametrize("dim,m,blocks,nt,nmax", [(2, 15, (2, 2), 40, 7), (2, 11, (3, 3), 30, 6),
                                                  (3, 5, (2, 2, 2), 24, 5)])
def test_greedy_selection_rule_recomputed(orc, dim, m, blocks, nt, nmax):
    """or_greedy Steps 5-6 against the paper's definition recomputed in numpy: a wrong
    norm (L2 / max instead of L1), selected parameters not excluded, or ties broken
    high all change the selected sequence."""
    g = orc.Grid(dim, m, blocks)
    tr = 0.1 * 100 ** np.random.default_rng(100 + m).random((nt, g.Q))
    res = g.greedy(tr, nmax)
    assert res["n"] == nmax and res["n_rejected"] == 0 and res["selected"][0] == 0
    for N, (best, gap, top) in enumerate(_recompute_selection(dim, m, blocks, tr, res["W"],
                                                              res["selected"], res["n"]), start=1):
        if gap > 1e-10:
            assert res["selected"][N] == best, (N, res["selected"], best)
        else:   # a genuine near-tie: either candidate is the argmax to rounding
            assert res["selected"][N] not in res["selected"][:N]
        assert abs(res["indicator"][N - 1] - top) <= 1e-10 * top


def test_greedy_tie_goes_to_lowest_index(orc):
    """Exact ties (a training parameter listed twice gives bitwise-equal indicators):
    AMB-13 takes the lowest index.  Put a copy of the parameter the greedy picks second
    BEFORE it in the list: the copy (lower index) must be picked instead, and the
    later duplicate is then dependent (same snapshot) -- rejected if ever chosen."""
    g = orc.Grid(2, 13, (2, 2))
    tr = 0.1 * 100 ** np.random.default_rng(31).random((20, 4))
    r0 = g.greedy(tr, 3)
    s1 = int(r0["selected"][1])
    assert s1 >= 1
    tr2 = np.vstack([tr[:1], tr[s1:s1 + 1], tr[1:]])      # copy at index 1; the original moves to s1+1
    r1 = g.greedy(tr2, 3)
    assert r1["selected"][1] == 1, r1["selected"]
    assert np.array_equal(r1["W"][:, :2], r0["W"][:, :2])
    assert (s1 + 1) not in list(r1["selected"])


def test_greedy_linear_rhs_family(orc):
    """Fixed operator, f(phi) = sum_r phi_r f_r with R = 3 (affine right-hand side,
    PAPER.md:98-103): every snapshot is A^{-1} sum_r phi_r f_r, so the solution manifold
    is 3-dimensional -- the greedy stops at n = 3 with the rest rejected -- and
    a_N(phi) = A_N^{-1} sum_r phi_r f_{N,r} is linear in phi, so Step 6's argmax is the
    largest |.|_1 of a linear map over the listed phi (recomputed in numpy)."""
    m = 12
    g = orc.Grid(2, m, (2, 2))
    rng = np.random.default_rng(17)
    theta = np.array([1.0, 3.0, 0.5, 2.0])
    nt, R = 15, 3
    tr = np.tile(theta, (nt, 1))
    phi = rng.standard_normal((nt, R))
    terms = rng.standard_normal((R, g.N))
    res = g.greedy(tr, 6, phi_train=phi, terms=terms)
    assert res["n"] == R and res["n_rejected"] == nt - R
    A = refs.cellwise_fd(2, m, (2, 2), theta).tocsc()
    X = spla.spsolve(A, terms.T)                              # A^{-1} f_r, columns
    s = np.linalg.svd(res["W"].T @ np.linalg.qr(X)[0], compute_uv=False)
    assert s.min() > 1 - 1e-10                                # span W = span A^{-1} f_r
    assert np.abs(res["fnr"] - terms @ res["W"]).max() <= 1e-12 * np.abs(terms).max() * np.sqrt(g.N)
    for N, (best, gap, top) in enumerate(_recompute_selection(2, m, (2, 2), tr, res["W"], res["selected"],
                                                              res["n"], rhs=lambda t: phi[t] @ terms), start=1):
        assert gap > 1e-10 and res["selected"][N] == best
        assert abs(res["indicator"][N - 1] - top) <= 1e-10 * top


# --------------------------------------------------------------------------- plain CG (context solver)
@pytest.mark.parametrize("dim,m,blocks", [(2, 20, (3, 3)), (3, 7, (2, 2, 2))])
def test_cg_matches_scipy(orc, dim, m, blocks):
    """or_cg is textbook CG (the context baseline of PAPER.md:31, 417): the same
    iteration count as scipy.sparse.linalg.cg on the independently assembled matrix
    (+-1) and the same solution."""
    g = orc.Grid(dim, m, blocks)
    mu = rand_mu(g.Q, rng=np.random.default_rng(23))
    A = refs.cellwise_fd(dim, m, blocks, mu).tocsr()
    b = np.random.default_rng(24).standard_normal(g.N)
    count = [0]
    xs, info = spla.cg(A, b, rtol=1e-10, atol=0.0, maxiter=5000,
                       callback=lambda xk: count.__setitem__(0, count[0] + 1))
    assert info == 0
    out = g.cg(mu, b=b, tol=1e-10)
    assert out["status"] == "CONVERGED" and abs(out["its"] - count[0]) <= 1
    xd = spla.spsolve(A.tocsc(), b)
    assert np.linalg.norm(out["x"] - xd) <= 1e-8 * np.linalg.norm(xd)
    assert np.linalg.norm(b - A @ out["x"]) <= 1e-10 * np.linalg.norm(b)


def test_nonfinite_rhs_is_reported(orc, small2d):
    """AMB-11: a NaN / Inf right-hand side is NONFINITE, not the f = 0
    shortcut (a NaN norm fails every comparison, so the finiteness test comes first)."""
    g, tr, res = small2d
    for bad in (np.nan, np.inf, -np.inf):
        b = np.ones(g.N)
        b[5] = bad
        for solve in (g.rbcg, g.rbi):
            out = solve(res["W"], res["ANq"], res["fn"], tr[0], b=b, max_iter=50)
            assert out["status"] == "NONFINITE" and out["its"] == 0, (bad, solve)
    out = g.rbcg(res["W"], res["ANq"], res["fn"], tr[0], b=np.zeros(g.N))
    assert out["status"] == "CONVERGED" and out["its"] == 0 and not np.any(out["x"])


def test_offline_blocks_blas_equals_plain(orc, small2d):
    """The full-size helper (or_apply_A per column + a BLAS matmul) equals or_offline_blocks."""
    g, _, res = small2d
    A1, f1 = g.offline_blocks(res["W"])
    A2, f2 = orc.offline_blocks_blas(g, res["W"])
    assert np.abs(A1 - A2).max() <= 1e-13 * np.abs(A1).max() and np.abs(f1 - f2).max() <= 1e-13 * np.abs(f1).max()
    for q in range(g.Q):
        assert np.array_equal(A2[q], A2[q].T)


@pytest.mark.parametrize("dim,mc,mf", [(2, 7, 31), (3, 3, 15)])
def test_fullsize_basis_interpolates_linearly(orc, dim, mc, mf):
    """The input recipe's prolongation reproduces a linear field exactly at fine nodes that
    are not next to the boundary ramp, and the result is orthonormal."""
    v = np.arange(1, mc + 1, dtype=float)
    f = v.copy()
    for ax in range(1, dim):
        f = f[..., None] * np.ones(mc)
    fine = f
    for ax in range(dim):
        fine = orc._interp_axis(fine, ax, mc, mf)
    hc, hf = 1.0 / (mc + 1), 1.0 / (mf + 1)
    xf = np.arange(1, mf + 1) * hf / hc                    # coarse index coordinate
    exp = np.where(xf <= mc, xf, mc * (mc + 1 - xf))       # linear, then the ramp to the zero boundary
    sl = (slice(None),) + (slice(4, 5),) * (dim - 1)
    got = fine[sl].reshape(-1)
    assert np.abs(got - exp).max() <= 1e-12
    g = orc.Grid(dim, mf, (2,) * dim)
    tr = 0.1 * 100 ** np.random.default_rng(3).random((12, g.Q))
    W, A, fn = orc.fullsize_basis(dim, mf, (2,) * dim, tr, 3, mc)
    assert np.abs(W.T @ W - np.eye(3)).max() < 1e-12
    A2, f2 = g.offline_blocks(W)
    assert np.abs(A - A2).max() <= 1e-12 * np.abs(A2).max()


# --------------------------------------------------------------------------- NEXT(3) variants
@pytest.mark.parametrize("dim,m,blocks", [(2, 7, (2, 2)), (3, 4, (2, 2, 2))])
def test_lexicographic_gs_is_textbook(orc, dim, m, blocks):
    """Lexicographic Gauss-Seidel (the comparison ordering): one forward sweep
    is (D + L) y_new = b - U y_old on the independently assembled matrix; the symmetric
    sweep adds the backward sweep (D + U) y = b - L y_fwd."""
    g = orc.Grid(dim, m, blocks)
    mu = rand_mu(g.Q)
    A = refs.cellwise_fd(dim, m, blocks, mu).tocsr()
    rng = np.random.default_rng(41)
    b, y0 = rng.standard_normal(g.N), rng.standard_normal(g.N)
    Lw, Up = sp_tril(A), sp_triu(A)
    yf = spla.spsolve_triangular(Lw, b - (A - Lw) @ y0, lower=True)
    yb = spla.spsolve_triangular(Up, b - (A - Up) @ yf, lower=False)
    assert np.abs(g.smooth(mu, b, y0, kind=orc.FWD_LEX) - yf).max() <= 1e-12 * np.abs(yf).max()
    assert np.abs(g.smooth(mu, b, y0, kind=orc.SYM_LEX) - yb).max() <= 1e-12 * np.abs(yb).max()


def sp_tril(A):
    import scipy.sparse as sp
    return sp.tril(A, format="csr")


def sp_triu(A):
    import scipy.sparse as sp
    return sp.triu(A, format="csr")


def _twolevel_independent(A, W, r, order):
    """M^{-1} r of the symmetric two-level RBI from independent pieces: the symmetric
    red-black GS from zero as explicit triangular solves (refs.sgs_rb_apply = B r), the
    Galerkin coarse correction C = W (W^T A W)^{-1} W^T by numpy:
    y1 = B r, y2 = y1 + C (r - A y1), y = y2 + B (r - A y2)."""
    C = lambda v: W @ np.linalg.solve(W.T @ (A @ W), W.T @ v)
    y1 = refs.sgs_rb_apply(A, order, r)
    y2 = y1 + C(r - A @ y1)
    return y2 + refs.sgs_rb_apply(A, order, r - A @ y2)


def test_symmetric_twolevel_preconditioner(orc, small2d):
    """NEXT(3): pre-smoothing with the adjoint sweep + coarse
    correction + post-smoothing equals the independent composition, and its matrix is
    symmetric positive definite -- unlike the paper's post-smoothed RBI, whose matrix is
    not symmetric (AMB-6)."""
    g, _, res = small2d
    W, ANq = res["W"], res["ANq"]
    mu = rand_mu(g.Q)
    A = refs.cellwise_fd(2, g.m, g.blocks, mu).tocsr()
    order = refs.red_black_order(2, g.m)
    r = np.random.default_rng(43).standard_normal(g.N)
    y = g.precond_apply(W, ANq, mu, r, precond=orc.PRECOND_SYM)
    ref = _twolevel_independent(A, W, r, order)
    assert np.linalg.norm(y - ref) <= 1e-11 * np.linalg.norm(ref)
    E = np.eye(g.N)
    Ms = np.stack([g.precond_apply(W, ANq, mu, E[:, j], precond=orc.PRECOND_SYM) for j in range(g.N)], 1)
    Mp = np.stack([g.precond_apply(W, ANq, mu, E[:, j], precond=orc.PRECOND_POST) for j in range(g.N)], 1)
    assert np.abs(Ms - Ms.T).max() <= 1e-11 * np.abs(Ms).max()
    assert np.linalg.eigvalsh(0.5 * (Ms + Ms.T)).min() > 0
    assert np.abs(Mp - Mp.T).max() > 1e-3 * np.abs(Mp).max()       # the paper's variant is not symmetric
    # forward red-black sweeps: pre (B,R) is the adjoint of post (R,B) -> symmetric as well
    Mf = np.stack([g.precond_apply(W, ANq, mu, E[:, j], smoother=orc.FWD_RBGS, precond=orc.PRECOND_SYM)
                   for j in range(g.N)], 1)
    assert np.abs(Mf - Mf.T).max() <= 1e-11 * np.abs(Mf).max()


def test_rbcg_symmetric_precond_is_textbook_pcg(orc, small2d):
    """RBCG with the symmetric two-level preconditioner is textbook PCG with M^{-1} built
    from independent pieces (scipy cg): the same iteration count +-1, the same solution."""
    g, _, res = small2d
    mu = rand_mu(g.Q, rng=np.random.default_rng(44))
    A = refs.cellwise_fd(2, g.m, g.blocks, mu).tocsr()
    order = refs.red_black_order(2, g.m)
    M = spla.LinearOperator(A.shape, matvec=lambda v: _twolevel_independent(A, res["W"], v, order))
    count = [0]
    b = np.ones(g.N)
    xs, info = spla.cg(A, b, M=M, rtol=1e-10, atol=0.0, maxiter=2000,
                       callback=lambda xk: count.__setitem__(0, count[0] + 1))
    out = g.rbcg(res["W"], res["ANq"], res["fn"], mu, precond=orc.PRECOND_SYM)
    assert out["status"] == "CONVERGED" and abs(out["its"] - count[0]) <= 1
    assert np.linalg.norm(out["x"] - xs) <= 1e-8 * np.linalg.norm(xs)


def test_rbcg_polak_ribiere(orc, small2d):
    """Polak-Ribiere beta (flexible CG, NEXT(3)): (1) with the symmetric preconditioner PR
    and the printed beta coincide in exact arithmetic (y_{k+1}^T r_k = 0), so the runs agree
    to rounding; (2) with the paper's preconditioner the oracle's run equals a textbook
    flexible PCG (PR beta) in numpy around the same preconditioner (a black box)."""
    g, _, res = small2d
    W, ANq, fn = res["W"], res["ANq"], res["fn"]
    mu = rand_mu(g.Q, rng=np.random.default_rng(45))
    a = g.rbcg(W, ANq, fn, mu, precond=orc.PRECOND_SYM, beta_rule=orc.BETA_FR, tol=1e-10)
    b = g.rbcg(W, ANq, fn, mu, precond=orc.PRECOND_SYM, beta_rule=orc.BETA_PR, tol=1e-10)
    assert abs(a["its"] - b["its"]) <= 1 and np.linalg.norm(a["x"] - b["x"]) <= 1e-9 * np.linalg.norm(a["x"])
    A = refs.cellwise_fd(2, g.m, g.blocks, mu).tocsr()
    Minv = lambda v: g.precond_apply(W, ANq, mu, v)
    f = np.ones(g.N)
    x, r = np.zeros(g.N), f.copy()
    y = Minv(r)
    p, rho, k = y.copy(), r @ y, 0
    while True:
        q = A @ p
        al = rho / (p @ q)
        x, r_old, r = x + al * p, r, r - al * q
        k += 1
        if np.linalg.norm(r) / np.linalg.norm(f) < 1e-10:
            break
        y = Minv(r)
        rho_new = y @ r
        p, rho = y + ((rho_new - y @ r_old) / rho) * p, rho_new
    c = g.rbcg(W, ANq, fn, mu, beta_rule=orc.BETA_PR)
    assert c["status"] == "CONVERGED" and abs(c["its"] - k) <= 1
    assert np.linalg.norm(c["x"] - x) <= 1e-9 * np.linalg.norm(x)
