"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Same seeded inputs (synth/), same basis (built by the oracle).  Criteria
(BASELINE.json north_star):
  iterations |d its| <= 1, ||x_gpu - x_or|| / ||x_or|| <= 1e-9,
  reduced coefficients a_n to relative 1e-10, residual histories to 1e-6
  relative (+1e-13 absolute rounding floor) at every common k.
"""
import os

import numpy as np
import pytest

from synth import CONFIGS, query_set, train_set

pytestmark = pytest.mark.gpu

X_TOL, A_TOL, H_TOL, H_ABS = 1e-9, 1e-10, 1e-6, 1e-13


@pytest.fixture(scope="module")
def rbs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1804_06363_b200 import build
    build.build()
    import paper_1804_06363_b200 as r
    return r


_BASES = {}


def oracle_basis(orc, dim, m, blocks, n, n_train, seed):
    key = (dim, m, tuple(blocks), n, n_train, seed)
    if key not in _BASES:
        g = orc.Grid(dim, m, blocks)
        rng = np.random.default_rng(seed)
        tr = 0.1 * 100 ** rng.random((n_train, g.Q))
        _BASES[key] = (g, g.greedy(tr, n))
    return _BASES[key]


def c1_basis(orc):
    c = CONFIGS["c1"]
    key = ("c1",)
    if key not in _BASES:
        g = orc.Grid(c.dim, c.m, c.blocks)
        _BASES[key] = (g, g.greedy(train_set(c), c.n))
    return _BASES[key]


def oracle_refs(g_or, W, ANq, fn, mus, method, **kw):
    """oracle solves of every mu, in threads (ctypes releases the GIL in the C oracle)."""
    from concurrent.futures import ThreadPoolExecutor
    solve = g_or.rbcg if method == "rbcg" else g_or.rbi
    with ThreadPoolExecutor(max(1, min(len(mus), os.cpu_count() or 1))) as ex:
        return list(ex.map(lambda mu: solve(W, ANq, fn, mu, **kw), list(mus)))


def compare(gout, g_or, W, ANq, fn, mus, method, check_hist=True, refs=None, **kw):
    """run the oracle on each mu (or take its precomputed results `refs`) and compare
    with the GPU result dict."""
    X = gout["X"].cpu().numpy()
    worst = dict(x=0.0, a=0.0, h=0.0, dits=0)
    for b, mu in enumerate(mus):
        solve = g_or.rbcg if method == "rbcg" else g_or.rbi
        ref = refs[b] if refs is not None else solve(W, ANq, fn, mu, **kw)
        assert gout["status"][b] == ref["status"], (b, gout["status"][b], ref["status"])
        d = abs(int(gout["its"][b]) - ref["its"])
        assert d <= 1, (b, gout["its"][b], ref["its"])
        xr = ref["x"]
        ex = np.linalg.norm(X[b] - xr) / max(np.linalg.norm(xr), 1e-300)
        assert ex <= X_TOL, (b, ex)
        if W is not None and W.shape[1] > 0 and gout.get("a_n") is not None:
            ea = np.abs(gout["a_n"][b] - ref["a_n"]).max() / np.abs(ref["a_n"]).max()
            assert ea <= A_TOL, (b, ea)
            worst["a"] = max(worst["a"], ea)
        if check_hist and "history" in gout:
            hg, hr = gout["history"][b], ref["hist"]
            k = min(len(hg), len(hr))
            dh = np.abs(hg[:k] - hr[:k])
            # relative 1e-6, plus an absolute floor: a recomputed residual b - A x
            # near 1e-10 carries rounding ~ eps ||A|| ||x|| / ||b||
            assert np.all(dh <= H_TOL * np.abs(hr[:k]) + H_ABS), (b, np.max(dh - H_TOL * np.abs(hr[:k])))
            eh = np.max(dh / np.maximum(np.abs(hr[:k]), 1e-300))
            worst["h"] = max(worst["h"], eh)
        worst["x"] = max(worst["x"], ex)
        worst["dits"] = max(worst["dits"], d)
    return worst


# ----------------------------------------------------------------------------- offline blocks
@pytest.mark.parametrize("dim,m,blocks,n", [(2, 37, (3, 3), 12), (3, 11, (2, 2, 2), 10),
                                            (2, 63, (2, 2), 16)])
def test_offline_blocks_on_device(orc, rbs, dim, m, blocks, n):
    g, res = oracle_basis(orc, dim, m, blocks, n, 30, 1)
    s = rbs.Solver(dim, m, blocks).load_basis(res["W"])  # blocks computed on the GPU
    A, f = s.offline_blocks()
    assert np.abs(A - res["ANq"]).max() <= 1e-12 * np.abs(res["ANq"]).max()
    assert np.abs(f - res["fn"]).max() <= 1e-12 * np.abs(res["fn"]).max()
    for q in range(g.Q):
        assert np.array_equal(A[q], A[q].T)


# ----------------------------------------------------------------------------- c1 in full
@pytest.mark.parametrize("method", ["rbcg", "rbi"])
def test_c1_all_queries(orc, rbs, method):
    c = CONFIGS["c1"]
    g, res = c1_basis(orc)
    s = rbs.Solver(c.dim, c.m, c.blocks).load_basis(res["W"], res["ANq"], res["fn"])
    mus = query_set(c)
    kw = dict(method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI,
              max_iter=20000 if method == "rbcg" else 500000, record_history=1)
    out = s.solve_batch(mus, **kw)
    assert all(st == "CONVERGED" for st in out["status"])
    assert np.all(out["true_relres"] < 1e-10 * 1.5)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, method,
            max_iter=kw["max_iter"])


@pytest.mark.parametrize("smoother,sweeps", [(1, 1), (0, 2), (1, 3)])
def test_c1_smoother_variants(orc, rbs, smoother, sweeps):
    c = CONFIGS["c1"]
    g, res = c1_basis(orc)
    s = rbs.Solver(c.dim, c.m, c.blocks).load_basis(res["W"], res["ANq"], res["fn"])
    mus = query_set(c)[:4]
    out = s.solve_batch(mus, smoother=smoother, sweeps=sweeps, record_history=1)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbcg", smoother=smoother,
            sweeps=sweeps)


# ----------------------------------------------------------------------------- ragged shapes
@pytest.mark.parametrize("dim,m,blocks,n,B", [
    (2, 37, (3, 3), 12, 5),      # ragged N (1369 = 4*342+1), npad 16, Bp 8
    (2, 50, (2, 3), 9, 13),      # rectangular block layout, Bp 16
    (3, 11, (2, 2, 2), 10, 3),   # 3D, N = 1331
    (3, 9, (2, 2, 2), 8, 33),    # 3D, B = 33 -> Bp 64
    (2, 47, (3, 3), 60, 64),     # 2D, npad 64, B = 64 -> two 32-query sub-batches
    (2, 63, (3, 3), 40, 32),     # 2D, the bench's n/B pair on a multi-strip grid
])
@pytest.mark.parametrize("method", ["rbcg", "rbi"])
def test_ragged_parity(orc, rbs, dim, m, blocks, n, B, method):
    g, res = oracle_basis(orc, dim, m, blocks, n, max(30, n + 20), 2)
    s = rbs.Solver(dim, m, blocks).load_basis(res["W"], res["ANq"], res["fn"])
    rng = np.random.default_rng(100 + B)
    mus = 0.1 * 100 ** rng.random((B, g.Q))
    mi = 20000 if method == "rbcg" else 500000
    out = s.solve_batch(mus, method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI,
                        max_iter=mi, record_history=1)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, method, max_iter=mi)


def test_fixed_iteration_mode(orc, rbs):
    """tol = 0, max_iter = K: x_K parity separates drift from threshold flips."""
    g, res = oracle_basis(orc, 2, 45, (3, 3), 10, 30, 3)
    s = rbs.Solver(2, 45, (3, 3)).load_basis(res["W"], res["ANq"], res["fn"])
    mus = 0.1 * 100 ** np.random.default_rng(4).random((8, 9))
    for method, K in (("rbcg", 25), ("rbi", 40)):
        out = s.solve_batch(mus, method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI,
                            tol=0.0, max_iter=K, record_history=1)
        assert all(st == "MAXIT" for st in out["status"]) and np.all(out["its"] == K)
        compare(out, g, res["W"], res["ANq"], res["fn"], mus, method, tol=0.0, max_iter=K)


# ----------------------------------------------------------------------------- paper lemmas on GPU
def test_lemma1_one_iteration(orc, rbs):
    import torch
    g, res = oracle_basis(orc, 2, 40, (2, 2), 8, 30, 5)
    W = res["W"]
    s = rbs.Solver(2, 40, (2, 2)).load_basis(W, res["ANq"], res["fn"])
    rng = np.random.default_rng(6)
    mus = 0.1 * 100 ** rng.random((4, 4))
    C = rng.standard_normal((4, W.shape[1]))
    rhs = np.stack([g.apply_A(mus[b], W @ C[b]) for b in range(4)])
    rt = torch.tensor(rhs, device="cuda")
    for method in (rbs.RBS_RBCG, rbs.RBS_RBI):
        out = s.solve_batch(mus, rhs=rt, method=method)
        assert np.all(out["its"] == 1) and all(st == "CONVERGED" for st in out["status"])
        X = out["X"].cpu().numpy()
        for b in range(4):
            assert np.linalg.norm(X[b] - W @ C[b]) <= 1e-10 * np.linalg.norm(W @ C[b])
            assert np.abs(out["a_n"][b] - C[b]).max() <= 1e-10 * np.abs(C[b]).max()


def test_lemma2_no_smoother(orc, rbs):
    g, res = oracle_basis(orc, 2, 40, (2, 2), 8, 30, 5)
    s = rbs.Solver(2, 40, (2, 2)).load_basis(res["W"], res["ANq"], res["fn"])
    mus = 0.1 * 100 ** np.random.default_rng(7).random((3, 4))
    out = s.solve_batch(mus, method=rbs.RBS_RBI, sweeps=0, max_iter=5)
    X = out["X"].cpu().numpy()
    for b in range(3):
        xhat = res["W"] @ orc.rb_solve(res["ANq"], res["fn"], mus[b])[0]
        assert out["status"][b] == "MAXIT"
        assert np.linalg.norm(X[b] - xhat) <= 1e-12 * np.linalg.norm(xhat)
    out = s.solve_batch(mus, method=rbs.RBS_RBCG, sweeps=0)
    assert all(st == "PRECOND" for st in out["status"]) and np.all(out["its"] == 1)


def test_empty_basis_is_sgs_pcg(orc, rbs):
    g = orc.Grid(2, 33, (3, 3))
    s = rbs.Solver(2, 33, (3, 3)).load_basis(np.zeros((g.N, 0)))
    mus = 0.1 * 100 ** np.random.default_rng(8).random((4, 9))
    out = s.solve_batch(mus, record_history=1, want_a_n=False)
    compare(out, g, None, None, None, mus, "rbcg")


def test_not_spd_query_does_not_fail_batch(orc, rbs):
    g, res = oracle_basis(orc, 2, 30, (2, 2), 6, 30, 9)
    s = rbs.Solver(2, 30, (2, 2)).load_basis(res["W"], res["ANq"], res["fn"])
    mus = np.array([[1.0, 2.0, 3.0, 4.0], [-5.0, -1.0, -2.0, -3.0], [0.5, 0.5, 2.0, 1.0]])
    out = s.solve_batch(mus)
    assert out["status"][1] == "REDUCED_NOT_SPD"
    assert out["status"][0] == "CONVERGED" and out["status"][2] == "CONVERGED"
    compare(dict(out, X=out["X"][[0, 2]], status=[out["status"][0], out["status"][2]],
                 its=out["its"][[0, 2]], a_n=out["a_n"][[0, 2]]),
            g, res["W"], res["ANq"], res["fn"], mus[[0, 2]], "rbcg", check_hist=False)


# ----------------------------------------------------------------------------- API behaviour
def test_host_output_determinism_and_launches(orc, rbs):
    c = CONFIGS["c1"]
    g, res = c1_basis(orc)
    s = rbs.Solver(c.dim, c.m, c.blocks).load_basis(res["W"], res["ANq"], res["fn"])
    mus = query_set(c)
    a = s.solve_batch(mus)
    b = s.solve_batch(mus)
    h = s.solve_batch(mus, x_location=rbs.RBS_MEM_HOST)
    assert a["launches"] > 0
    assert np.array_equal(a["X"].cpu().numpy(), b["X"].cpu().numpy())  # bitwise run to run
    assert np.array_equal(a["X"].cpu().numpy(), h["X"].numpy())
    assert np.array_equal(a["its"], h["its"])


def test_errors_are_status_codes(rbs):
    import ctypes as C
    s = rbs.Solver(2, 20, (2, 2))
    with pytest.raises(rbs.RbsError, match="E_STATE"):
        s.solve_batch(np.ones((2, 4)))  # no basis yet
    with pytest.raises(rbs.RbsError, match="E_DIM"):
        rbs.rbs_set_operator_blocks(s.ctx, 4, 10, (2, 2))
    s.load_basis(np.linalg.qr(np.random.default_rng(0).standard_normal((400, 3)))[0])
    with pytest.raises(rbs.RbsError, match="E_DIM"):
        s.solve_batch(np.ones((65, 4)))
    assert rbs.lib().rbs_last_error(s.ctx).decode()


# ----------------------------------------------------------------------------- GPU greedy
def test_gpu_greedy_matches_oracle_c1(orc, rbs):
    c = CONFIGS["c1"]
    g, res = c1_basis(orc)
    s = rbs.Solver(c.dim, c.m, c.blocks)
    gr = s.build_greedy(train_set(c), c.n)
    assert gr["n"] == res["n"] and gr["n_rejected"] == res["n_rejected"]
    sel_g, sel_o = list(gr["selected"]), list(res["selected"])
    if sel_g != sel_o:  # allowed only at a genuine near-tie of the oracle indicator
        k = next(i for i in range(len(sel_o)) if sel_g[i] != sel_o[i])
        assert abs(gr["indicator"][k - 1] - res["indicator"][k - 1]) <= 1e-10 * res["indicator"][k - 1]
    else:
        Wg = gr["W"].cpu().numpy()
        sv = np.linalg.svd(Wg.T @ res["W"], compute_uv=False)
        assert sv.min() >= 1 - 1e-8  # principal angles <= ~1e-4 rad (cos >= 1-1e-8)
        assert np.abs(gr["indicator"] - res["indicator"]).max() <= 1e-8 * np.abs(res["indicator"]).max()
        assert np.all(np.abs(gr["snap_iters"] - res["snap_iters"]) <= 1)


def test_gpu_greedy_basis_solves(orc, rbs):
    g, res = oracle_basis(orc, 3, 9, (2, 2, 2), 8, 25, 11)
    s = rbs.Solver(3, 9, (2, 2, 2))
    rng = np.random.default_rng(11)
    tr = 0.1 * 100 ** rng.random((25, 8))
    gr = s.build_greedy(tr, 8)
    Wg = gr["W"].cpu().numpy()
    assert np.abs(Wg.T @ Wg - np.eye(gr["n"])).max() < 1e-12
    assert list(gr["selected"]) == list(res["selected"])
    mus = 0.1 * 100 ** rng.random((4, 8))
    out = s.solve_batch(mus, record_history=1)
    # the oracle solves with the oracle's own basis; same subspace => same iterates
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbcg")


# ----------------------------------------------------------------------------- full size (c2)
def test_c2_full_size_sampled(orc, rbs):
    """BASELINE configs[1] at full size in bench.py's launch configuration (B = 32):
    oracle-built basis (coarse greedy interpolated, DESIGN.md input recipe);
    sampled outputs the oracle computes one by one + a property at any size."""
    c = CONFIGS["c2"]
    W, ANq, fn = orc.interpolated_basis(c.dim, c.m, c.blocks, train_set(c), c.n, 63)
    g = orc.Grid(c.dim, c.m, c.blocks)
    s = rbs.Solver(c.dim, c.m, c.blocks).load_basis(W, ANq, fn)
    mus = query_set(c)[:c.B]
    # (1) fixed-iteration mode on the whole batch, oracle on 3 sampled queries
    out = s.solve_batch(mus, tol=0.0, max_iter=30, record_history=1)
    idx = [0, 13, 31]
    compare(dict(out, X=out["X"][idx], status=[out["status"][i] for i in idx], its=out["its"][idx],
                 a_n=out["a_n"][idx], history=[out["history"][i] for i in idx]),
            g, W, ANq, fn, mus[idx], "rbcg", tol=0.0, max_iter=30)
    # (2) converged batch: the recurrence residual met the tolerance (Step 8);
    #     the true residual of every returned x, recomputed with the oracle's
    #     operator, matches the GPU's reported true_relres (the recurrence and
    #     true residuals drift apart by up to ~2x at 1e-10 with the paper's
    #     non-symmetric preconditioner -- the oracle shows the same); one query
    #     is compared in full
    out = s.solve_batch(mus, record_history=1)
    assert all(st == "CONVERGED" for st in out["status"]) and np.all(out["relres"] < 1e-10)
    X = out["X"].cpu().numpy()
    for b in range(c.B):
        t = np.linalg.norm(1.0 - g.apply_A(mus[b], X[b])) / np.sqrt(g.N)
        assert abs(t - out["true_relres"][b]) <= 1e-3 * t + 1e-13, b
        assert t < 1e-9, b
    idx = [0, 5, 9, 13, 18, 22, 27, 31]       # 8 of the 32, in full at convergence
    refs = oracle_refs(g, W, ANq, fn, mus[idx], "rbcg")
    compare(dict(out, X=out["X"][idx], status=[out["status"][i] for i in idx], its=out["its"][idx],
                 a_n=out["a_n"][idx], history=[out["history"][i] for i in idx]),
            g, W, ANq, fn, mus[idx], "rbcg", refs=refs)


# ----------------------------------------------------------------------------- full size c3 / c4
def _full_size_sampled(orc, rbs, cname, n_basis, m_coarse, fixed_its, idx, true_floor=1e-7):
    """BASELINE configs[2] / configs[3] at full grid size in the config's batch
    size: a small-n oracle-built basis (coarse greedy interpolated, oracle MGS and
    offline blocks -- at n = 60 the oracle's fine-grid blocks alone take minutes),
    (1) fixed-iteration parity on sampled queries, (2) the converged batch: every
    returned x has a true residual below the tolerance band, recomputed by the
    oracle's operator, matching the GPU's reported true_relres."""
    c = CONFIGS[cname]
    W, ANq, fn = orc.interpolated_basis(c.dim, c.m, c.blocks, train_set(c)[:64], n_basis, m_coarse)
    g = orc.Grid(c.dim, c.m, c.blocks)
    s = rbs.Solver(c.dim, c.m, c.blocks).load_basis(W, ANq, fn)
    mus = query_set(c)[:c.B]
    out = s.solve_batch(mus, tol=0.0, max_iter=fixed_its, record_history=1)
    compare(dict(out, X=out["X"][idx], status=[out["status"][i] for i in idx], its=out["its"][idx],
                 a_n=out["a_n"][idx], history=[out["history"][i] for i in idx]),
            g, W, ANq, fn, mus[idx], "rbcg", tol=0.0, max_iter=fixed_its)
    out = s.solve_batch(mus)
    assert all(st == "CONVERGED" for st in out["status"]) and np.all(out["relres"] < 1e-10)
    X = out["X"].cpu().numpy()
    fnorm = np.sqrt(g.N)
    for b in range(len(mus)):
        t = np.linalg.norm(1.0 - g.apply_A(mus[b], X[b])) / fnorm
        assert abs(t - out["true_relres"][b]) <= 1e-3 * t + 1e-13, b
        # the stop test is on the recurrence residual (Step 8, AMB-7); in fp64 the
        # true residual of CG floors near eps * cond(A) (here ~1e-16 * 4e8 at
        # h = 1/2048 with a 100x coefficient contrast), so it is bounded, not 1e-10
        assert t < true_floor, (b, t)
    return out


def test_c3_full_size_sampled(orc, rbs):
    """c3: 2D 2047^2 (N = 4.19M), 3x3 blocks, B = 64 (two 32-query row-march passes)."""
    out = _full_size_sampled(orc, rbs, "c3", 8, 63, 10, [0, 37, 63])
    assert len(out["its"]) == 64


def test_c4_full_size_sampled(orc, rbs):
    """c4: 3D 255^3 (N = 16.6M), 2x2x2 blocks, B = 16."""
    out = _full_size_sampled(orc, rbs, "c4", 8, 31, 5, [0, 15])
    assert len(out["its"]) == 16


_FULL = {}


def _fullsize(orc, cname, m_coarse):
    """full-size input at the bench's RB dimension (oracle.fullsize_basis: coarse oracle
    greedy, interpolated, orthonormalised, oracle offline blocks); built once per session"""
    if cname not in _FULL:
        c = CONFIGS[cname]
        _FULL[cname] = orc.fullsize_basis(c.dim, c.m, c.blocks, train_set(c), c.n, m_coarse,
                                          threads=os.cpu_count() or 1)
    return _FULL[cname]


def _n_full_fixed(orc, rbs, cname, m_coarse, idx, K):
    """BASELINE configs at full size AND the bench's n (npad 64 kernels, the explicit
    A_n^{-1}): K fixed RBCG iterations of the config's batch (tol = 0), the oracle on
    sampled queries."""
    c = CONFIGS[cname]
    W, ANq, fn = _fullsize(orc, cname, m_coarse)
    assert W.shape[1] == c.n
    g = orc.Grid(c.dim, c.m, c.blocks)
    s = rbs.Solver(c.dim, c.m, c.blocks).load_basis(W, ANq, fn)
    mus = query_set(c)[:c.B]
    out = s.solve_batch(mus, tol=0.0, max_iter=K, record_history=1)
    assert all(st == "MAXIT" for st in out["status"]) and np.all(out["its"] == K)
    refs = oracle_refs(g, W, ANq, fn, mus[idx], "rbcg", tol=0.0, max_iter=K)
    return compare(dict(out, X=out["X"][idx], status=[out["status"][i] for i in idx], its=out["its"][idx],
                        a_n=out["a_n"][idx], history=[out["history"][i] for i in idx]),
                   g, W, ANq, fn, mus[idx], "rbcg", refs=refs, tol=0.0, max_iter=K)


def test_c3_full_size_n60(orc, rbs):
    """c3: 2047^2, n = 60, B = 64 (two 32-query passes), 20 fixed iterations, 3 queries."""
    _n_full_fixed(orc, rbs, "c3", 63, [0, 37, 63], 20)


def test_c4_full_size_n60(orc, rbs):
    """c4: 255^3, n = 60, B = 16, 20 fixed iterations, 2 queries."""
    _n_full_fixed(orc, rbs, "c4", 31, [0, 15], 20)


# ----------------------------------------------------------------------------- mesh slabs
@pytest.mark.parametrize("G", [2, 3])
def test_virtual_slabs_match_oracle_and_full_solve(orc, rbs, G):
    """Mesh-slab mode: G z-slabs with ghost planes, halo copies and
    fixed-order cross-slab partial sums give the oracle's RBCG (its +-1, x 1e-9,
    histories) and agree with the unpartitioned GPU solve to rounding."""
    dim, m, blocks, n = 3, 23, (2, 2, 2), 8
    g, res = oracle_basis(orc, dim, m, blocks, n, 30, 5)
    rng = np.random.default_rng(31 + G)
    mus = 0.1 * 100 ** rng.random((5, g.Q))
    full = rbs.Solver(dim, m, blocks).load_basis(res["W"], res["ANq"], res["fn"])
    ref_gpu = full.solve_batch(mus, record_history=1)
    s = rbs.Solver(dim, m, blocks).load_basis(res["W"], res["ANq"], res["fn"]).set_slabs(G)
    out = s.solve_batch(mus, record_history=1)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbcg")
    Xs, Xf = out["X"].cpu().numpy(), ref_gpu["X"].cpu().numpy()
    assert np.abs(Xs - Xf).max() <= 1e-9 * np.abs(Xf).max()
    assert np.all(np.abs(out["its"] - ref_gpu["its"]) <= 1)
    assert np.allclose(out["true_relres"], ref_gpu["true_relres"], rtol=1e-3, atol=1e-13)
    # fixed-iteration mode through the slab path
    fx = s.solve_batch(mus, tol=0.0, max_iter=7)
    compare(fx, g, res["W"], res["ANq"], res["fn"], mus, "rbcg", check_hist=False, tol=0.0, max_iter=7)


def test_virtual_slabs_errors(rbs):
    s2 = rbs.Solver(2, 15, (2, 2))
    with pytest.raises(rbs.RbsError):
        s2.set_slabs(2)                      # 2D: unsupported
    s3 = rbs.Solver(3, 11, (2, 2, 2))
    with pytest.raises(rbs.RbsError):
        s3.set_slabs(4)                      # 11 planes / 4 slabs < 4 planes each
    s3.set_slabs(2)
    s3.set_slabs(1)


def test_dist_slab_single_rank_nccl(orc, rbs):
    """Mesh slabs over ranks (rbs_dist_init) with one rank: the NCCL code path
    (column sums + allreduce before every scalar step, grouped send/recv with no
    neighbours, graph capture with NCCL calls) reproduces the oracle's RBCG.  The
    multi-rank partition itself is the virtual-slab test's (same passes, halos,
    partial columns); only the transport differs."""
    dim, m, blocks, n = 3, 19, (2, 2, 2), 8
    g, res = oracle_basis(orc, dim, m, blocks, n, 30, 6)
    rng = np.random.default_rng(77)
    mus = 0.1 * 100 ** rng.random((4, g.Q))
    s = rbs.Solver(dim, m, blocks).dist_init(rbs.rbs_nccl_unique_id(), 1, 0, 3)
    assert s.local["z0"] == 1 and s.local["z1"] == m + 1 and s.local["n_owned"] == g.N
    s.load_basis(res["W"], res["ANq"], res["fn"])
    out = s.solve_batch(mus, record_history=1)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbcg")


# ----------------------------------------------------------------------------- active RB dimension
@pytest.mark.parametrize("dim,m,blocks,n,na,B", [
    (2, 47, (3, 3), 24, 7, 9),       # fixed active dimension < n (iterations-vs-n study)
    (2, 63, (3, 3), 40, 40, 5),      # n_active = n: same as the full solve
    (3, 11, (2, 2, 2), 10, 4, 6),    # 3D flat kernels
])
@pytest.mark.parametrize("method", ["rbcg", "rbi"])
def test_fixed_active_dimension(orc, rbs, dim, m, blocks, n, na, B, method):
    """opts.n_active: leading-block reduced solves (DESIGN.md AMB-19) against the oracle."""
    g, res = oracle_basis(orc, dim, m, blocks, n, max(30, n + 20), 2)
    s = rbs.Solver(dim, m, blocks).load_basis(res["W"], res["ANq"], res["fn"])
    rng = np.random.default_rng(300 + na)
    mus = 0.1 * 100 ** rng.random((B, g.Q))
    mi = 20000 if method == "rbcg" else 500000
    out = s.solve_batch(mus, method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI,
                        max_iter=mi, record_history=1, n_active=na)
    assert np.all(out["n_active"] == na)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, method, max_iter=mi, n_active=na)


@pytest.mark.parametrize("dim,m,blocks,n,na0,gamma,B", [
    (2, 47, (3, 3), 24, 1, 3.0, 8),     # grows from 1 while the residual falls slowly
    (2, 63, (3, 3), 40, 5, 1.5, 40),    # two sub-batches; multi-strip grid
    (3, 11, (2, 2, 2), 10, 2, 4.0, 5),  # 3D
])
def test_adaptive_n_rule(orc, rbs, dim, m, blocks, n, na0, gamma, B):
    """opts.gamma: the adaptive-n rule of PAPER.md:287 (RBCG); the final active
    dimension of every query equals the oracle's trace, iterations/x/histories match."""
    g, res = oracle_basis(orc, dim, m, blocks, n, max(30, n + 20), 2)
    s = rbs.Solver(dim, m, blocks).load_basis(res["W"], res["ANq"], res["fn"])
    rng = np.random.default_rng(400 + B)
    mus = 0.1 * 100 ** rng.random((B, g.Q))
    out = s.solve_batch(mus, record_history=1, n_active=na0, gamma=gamma)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbcg", n_active=na0, gamma=gamma)
    grew = 0
    for b, mu in enumerate(mus):
        ref = g.rbcg(res["W"], res["ANq"], res["fn"], mu, n_active=na0, gamma=gamma)
        assert int(out["n_active"][b]) == int(ref["active_n"][-1]), (b, out["n_active"][b], ref["active_n"])
        grew += int(ref["active_n"][-1]) > na0
    assert grew > 0   # the rule actually fired


def test_active_dimension_errors(rbs):
    import paper_1804_06363_b200 as r
    s = rbs.Solver(2, 31, (2, 2)).load_basis(np.linalg.qr(np.random.default_rng(0).random((961, 6)))[0])
    mus = np.ones((2, 4))
    for kw in (dict(n_active=7), dict(n_active=-1), dict(gamma=-1.0), dict(method=r.RBS_RBI, gamma=2.0)):
        with pytest.raises(RuntimeError):
            s.solve_batch(mus, **kw)


# ----------------------------------------------------------------------------- Jacobi smoother
@pytest.mark.parametrize("dim,m,blocks,n,B,omega,sweeps,method", [
    (2, 37, (3, 3), 12, 5, 1.0, 1, "rbcg"),     # undamped, odd sweeps: prolongation into T
    (2, 47, (3, 3), 20, 8, 0.8, 2, "rbcg"),     # even sweeps
    (3, 11, (2, 2, 2), 10, 3, 0.8, 1, "rbcg"),  # 3D
    (2, 37, (3, 3), 12, 5, 0.8, 1, "rbi"),      # RBI: odd sweeps end in T -> copy
    (2, 31, (2, 2), 8, 9, 0.7, 2, "rbi"),
    (3, 9, (2, 2, 2), 8, 4, 0.8, 3, "rbi"),
])
def test_jacobi_smoother(orc, rbs, dim, m, blocks, n, B, omega, sweeps, method):
    """S = damped Jacobi ("the smoother (Jacobi or Gauss-Seidel)") in RBI and RBCG."""
    g, res = oracle_basis(orc, dim, m, blocks, n, max(30, n + 20), 2)
    s = rbs.Solver(dim, m, blocks).load_basis(res["W"], res["ANq"], res["fn"])
    rng = np.random.default_rng(500 + B)
    mus = 0.1 * 100 ** rng.random((B, g.Q))
    mi = 20000 if method == "rbcg" else 500000
    out = s.solve_batch(mus, method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI, max_iter=mi,
                        record_history=1, smoother=rbs.RBS_SMOOTH_JACOBI, sweeps=sweeps, omega=omega)
    assert all(st == "CONVERGED" for st in out["status"]), out["status"]
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, method, max_iter=mi, smoother=orc.JACOBI,
            sweeps=sweeps, omega=omega)


def test_jacobi_errors_and_graph_reuse(orc, rbs):
    """omega outside (0, 2) is an argument error; one Solver alternating smoothers and
    active dimensions rebuilds its iteration graph (results equal fresh solves)."""
    g, res = oracle_basis(orc, 2, 31, (2, 2), 8, 30, 2)
    s = rbs.Solver(2, 31, (2, 2)).load_basis(res["W"], res["ANq"], res["fn"])
    mus = 0.1 * 100 ** np.random.default_rng(7).random((3, g.Q))
    for om in (0.0, 2.0, -1.0):
        with pytest.raises(RuntimeError):
            s.solve_batch(mus, smoother=rbs.RBS_SMOOTH_JACOBI, omega=om)
    a = s.solve_batch(mus)
    b = s.solve_batch(mus, smoother=rbs.RBS_SMOOTH_JACOBI, omega=0.9)
    c = s.solve_batch(mus, n_active=3)
    d = s.solve_batch(mus)
    assert np.array_equal(a["X"].cpu().numpy(), d["X"].cpu().numpy())
    for out, kw in ((b, dict(smoother=orc.JACOBI, omega=0.9)), (c, dict(n_active=3))):
        compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbcg", check_hist=False, **kw)


@pytest.mark.parametrize("smoother,sweeps", [(0, 2), (1, 3)])
def test_rbi_many_half_sweeps_flat_path(orc, rbs, smoother, sweeps):
    """RBI on a 2D grid with more half-sweeps than the row march holds (flat kernels)."""
    c = CONFIGS["c1"]
    g, res = c1_basis(orc)
    s = rbs.Solver(c.dim, c.m, c.blocks).load_basis(res["W"], res["ANq"], res["fn"])
    mus = query_set(c)[:3]
    out = s.solve_batch(mus, method=rbs.RBS_RBI, max_iter=500000, smoother=smoother, sweeps=sweeps,
                        record_history=1)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbi", max_iter=500000, smoother=smoother,
            sweeps=sweeps)


def test_gpu_basis_from_samples_matches_oracle(orc, rbs):
    """RBS_GREEDY_SAMPLES (multi-fidelity fine half): select on a coarse grid
    (oracle greedy on 31^2), then build the fine basis from the selected parameters on the
    GPU; equals the oracle's or_basis_from_samples (same snapshots, MGS, offline blocks)."""
    dim, blocks, n = 2, (3, 3), 8
    gc = orc.Grid(dim, 31, blocks)
    rng = np.random.default_rng(31)
    tr = 0.1 * 100 ** rng.random((60, gc.Q))
    coarse = gc.greedy(tr, n)
    mus = tr[coarse["selected"]]
    gf = orc.Grid(dim, 63, blocks)
    ref = gf.basis_from_samples(mus)
    s = rbs.Solver(dim, 63, blocks)
    res = s.build_greedy(mus, n, samples=True)
    assert res["n"] == ref["n"] == n
    assert np.array_equal(res["selected"], np.arange(n))
    W = res["W"].cpu().numpy()
    assert np.abs(W - ref["W"]).max() <= 1e-8
    assert np.abs(res["ANq"] - ref["ANq"]).max() <= 1e-8 * np.abs(ref["ANq"]).max()
    assert np.abs(res["fn"] - ref["fn"]).max() <= 1e-8 * np.abs(ref["fn"]).max()


@pytest.mark.parametrize("dim,m,blocks,n", [(2, 63, (3, 3), 12), (3, 23, (2, 2, 2), 10)])
def test_gpu_batched_samples_match_oracle(orc, rbs, dim, m, blocks, n):
    """RBS_GREEDY_SAMPLES_BATCH (AMB-27): the same samples solved 8 at a time (RBCG with the
    symmetric two-level preconditioner on the basis so far) -- every snapshot is the fine
    solution to 1e-12, so the basis equals the oracle's or_basis_from_samples (same MGS
    order) to the snapshot tolerance, and so do the offline blocks."""
    gc = orc.Grid(dim, 15 if dim == 3 else 31, blocks)
    tr = 0.1 * 100 ** np.random.default_rng(32).random((60, gc.Q))
    mus = tr[gc.greedy(tr, n)["selected"]]
    ref = orc.Grid(dim, m, blocks).basis_from_samples(mus)
    res = rbs.Solver(dim, m, blocks).build_greedy(mus, n, samples=True, batched=True)
    assert res["n"] == ref["n"] == n and res["n_rejected"] == 0
    W = res["W"].cpu().numpy()
    assert np.abs(W - ref["W"]).max() <= 1e-7
    sv = np.linalg.svd(W.T @ ref["W"], compute_uv=False)
    assert sv.min() >= 1 - 1e-10
    assert np.abs(res["ANq"] - ref["ANq"]).max() <= 1e-7 * np.abs(ref["ANq"]).max()
    assert np.all(res["snap_iters"] > 0)


@pytest.mark.parametrize("dim,m,blocks,n,B", [
    (3, 13, (2, 2, 2), 20, 16),   # Bp 16: two rows per warp in the row-segment passes, k_wtr<16>
    (3, 12, (2, 3, 2), 24, 32),   # Bp 32: one row per warp, k_wtr<32>, ragged segments (12 = 3 x 4)
    (3, 10, (2, 2, 2), 60, 9),    # npad 64 with Bp 16 -> k_wtr with 32-node chunks
])
@pytest.mark.parametrize("method", ["rbcg", "rbi"])
def test_3d_row_segment_passes(orc, rbs, dim, m, blocks, n, B, method):
    """The 3D RBCG passes (k_pnew3 + k_sigma3r, k_xr3r + k_wtr, k_gs3r) and the RBI path
    against the oracle at the batch widths they specialise on."""
    g, res = oracle_basis(orc, dim, m, blocks, n, max(30, n + 20), 3)
    s = rbs.Solver(dim, m, blocks).load_basis(res["W"], res["ANq"], res["fn"])
    rng = np.random.default_rng(700 + B)
    mus = 0.1 * 100 ** rng.random((B, g.Q))
    mi = 20000 if method == "rbcg" else 500000
    out = s.solve_batch(mus, method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI,
                        max_iter=mi, record_history=1)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, method, max_iter=mi)
