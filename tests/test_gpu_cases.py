"""GPU parity for the general affine (face-coefficient) operator and the paper's
Case 1 / Case 2 problems (NEXT(4), DESIGN.md AMB-23): the CUDA path through the
C ABI against the oracle, on the same seeded inputs and the same basis."""
import numpy as np
import pytest

from synth import CONFIGS, query_set
from synth import cases
from test_gpu_parity import c1_basis, compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rbs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1804_06363_b200 import build
    build.build()
    import paper_1804_06363_b200 as r
    return r


def snapshot_basis(orc, g, P, mus, tol=1e-12):
    """oracle snapshots x(mu) = A(theta(mu))^-1 f(mu) (SGS-PCG), MGS, offline blocks."""
    W = None
    for mu in mus:
        x = g.rbcg(None, None, None, P["theta"](mu), b=P["phi"](mu) @ P["terms"], tol=tol)["x"]
        W, _ = orc.mgs_append(W, x)
    ANq, fn = g.offline_blocks(W)
    return W, ANq, fn


def test_faces_from_blocks_gpu_equals_block_path(orc, rbs):
    """c1 as a face operator (flat kernels) against the oracle and the block row-march path."""
    c = CONFIGS["c1"]
    g, res = c1_basis(orc)
    F = cases.faces_from_blocks(c.dim, c.m, c.blocks)
    sf = rbs.Solver(c.dim, c.m, faces=F).load_basis(res["W"], res["ANq"], res["fn"])
    sb = rbs.Solver(c.dim, c.m, c.blocks).load_basis(res["W"], res["ANq"], res["fn"])
    mus = query_set(c)
    for method in ("rbcg", "rbi"):
        kw = dict(method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI,
                  max_iter=20000 if method == "rbcg" else 500000, record_history=1)
        of, ob = sf.solve_batch(mus, **kw), sb.solve_batch(mus, **kw)
        compare(of, g, res["W"], res["ANq"], res["fn"], mus, method, max_iter=kw["max_iter"])
        assert np.all(np.abs(of["its"] - ob["its"]) <= 1)
        xf, xb = of["X"].cpu().numpy(), ob["X"].cpu().numpy()
        assert np.linalg.norm(xf - xb) <= 1e-9 * np.linalg.norm(xb)


def test_offline_blocks_from_faces_on_device(orc, rbs):
    dim, m = 3, 7
    P = cases.case_problem(2, m)
    g = orc.Grid(dim, m, faces=P["faces"])
    W, ANq, fn = snapshot_basis(orc, g, P, cases.case_params(2, 6, 11))
    s = rbs.Solver(dim, m, faces=P["faces"]).load_basis(W)     # blocks computed on the GPU
    A, f = s.offline_blocks()
    assert np.abs(A - ANq).max() <= 1e-12 * np.abs(ANq).max()
    assert np.abs(f - fn).max() <= 1e-12 * np.abs(fn).max()


def test_affine_rhs_kernel(rbs):
    m = 9
    P = cases.case_problem(2, m)
    s = rbs.Solver(3, m, faces=P["faces"])
    mus = cases.case_params(2, 7, 5)
    phi = np.stack([P["phi"](mu) for mu in mus])
    got = s.affine_rhs(phi, P["terms"]).cpu().numpy()
    ref = phi @ P["terms"]
    assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("case,m,n_train,B", [(1, 11, 6, 5), (2, 15, 10, 6)])
@pytest.mark.parametrize("method", ["rbcg", "rbi"])
def test_case_parity(orc, rbs, case, m, n_train, B, method):
    """Case 1 / Case 2: GPU solves with the device-assembled affine
    right-hand side against the oracle with f(mu) = sum_r phi_r(mu) f_r."""
    P = cases.case_problem(case, m)
    g = orc.Grid(3, m, faces=P["faces"])
    W, ANq, fn = snapshot_basis(orc, g, P, cases.case_params(case, n_train, 100 + case))
    s = rbs.Solver(3, m, faces=P["faces"]).load_basis(W, ANq, fn)
    mus = cases.case_params(case, B, 200 + case)
    th = np.stack([P["theta"](mu) for mu in mus])
    phi = np.stack([P["phi"](mu) for mu in mus])
    rhs = s.affine_rhs(phi, P["terms"])
    mi = 20000 if method == "rbcg" else 500000
    out = s.solve_batch(th, rhs=rhs, method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI,
                        max_iter=mi, record_history=1)
    assert all(st == "CONVERGED" for st in out["status"]), out["status"]
    X = out["X"].cpu().numpy()
    for b in range(B):
        ref = (g.rbcg if method == "rbcg" else g.rbi)(W, ANq, fn, th[b], b=phi[b] @ P["terms"], max_iter=mi)
        assert ref["status"] == "CONVERGED"
        assert abs(int(out["its"][b]) - ref["its"]) <= 1, (b, out["its"][b], ref["its"])
        assert np.linalg.norm(X[b] - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
        hg, hr = out["history"][b], ref["hist"]
        k = min(len(hg), len(hr))
        assert np.all(np.abs(hg[:k] - hr[:k]) <= 1e-6 * np.abs(hr[:k]) + 1e-13)


@pytest.mark.parametrize("case", [1, 2])
def test_gpu_greedy_affine_rhs(orc, rbs, case):
    """rbs_build_greedy_affine: orthonormal W; offline blocks equal the oracle's W^T A_q W;
    f_{N,r} = W^T f_r; every selected parameter is reproduced from span W (Lemma 1,
    PAPER.md:184-196: one RBCG iteration to the snapshot tolerance)."""
    import torch
    m, n_max = 11, 8
    P = cases.case_problem(case, m)
    g = orc.Grid(3, m, faces=P["faces"])
    mus = cases.case_params(case, 24, 300 + case)
    th = np.stack([P["theta"](mu) for mu in mus])
    phi = np.stack([P["phi"](mu) for mu in mus])
    s = rbs.Solver(3, m, faces=P["faces"])
    res = s.build_greedy(th, n_max, phi_train=phi, terms=P["terms"])
    n = res["n"]
    assert n == n_max
    W = res["W"].cpu().numpy()
    assert np.abs(W.T @ W - np.eye(n)).max() < 1e-12
    ANq, _ = g.offline_blocks(W)
    assert np.abs(res["ANq"] - ANq).max() <= 1e-11 * np.abs(ANq).max()
    assert np.abs(res["fn"] - P["terms"] @ W).max() <= 1e-11 * np.abs(res["fn"]).max()
    sel = res["selected"]
    assert sel[0] == 0 and len(set(sel.tolist())) == n
    rhs = s.affine_rhs(phi[sel], P["terms"])
    out = s.solve_batch(th[sel], rhs=rhs, tol=1e-9)
    assert np.all(out["its"] <= 1), out["its"]
    assert torch.isfinite(out["X"]).all()


@pytest.mark.parametrize("case", [1, 2])
def test_gpu_greedy_affine_matches_oracle(orc, rbs, case):
    """rbs_build_greedy_affine against the oracle greedy with the same affine right-hand
    sides (or_set_greedy_rhs): same selected parameters, basis, offline blocks, f_{N,r}."""
    m, n_max = 9, 6
    P = cases.case_problem(case, m)
    g = orc.Grid(3, m, faces=P["faces"])
    mus = cases.case_params(case, 16, 500 + case)
    th = np.stack([P["theta"](mu) for mu in mus])
    phi = np.stack([P["phi"](mu) for mu in mus])
    ref = g.greedy(th, n_max, phi_train=phi, terms=P["terms"])
    s = rbs.Solver(3, m, faces=P["faces"])
    res = s.build_greedy(th, n_max, phi_train=phi, terms=P["terms"])
    assert res["n"] == ref["n"]
    assert np.array_equal(res["selected"], ref["selected"]), (res["selected"], ref["selected"])
    # later columns come from nearly dependent snapshots (solved to 1e-12 by two solvers):
    # MGS amplifies their difference, so compare the spaces and the leading columns
    W = res["W"].cpu().numpy()
    assert np.abs(W[:, :2] - ref["W"][:, :2]).max() <= 1e-9
    Wr = ref["W"]
    # span(W_gpu) in span(W_oracle): the error of a column is the snapshot tolerance (1e-12)
    # times ||x|| / ||w|| of its MGS step (up to 1e10 by the drop rule; ~1e6 for the last
    # columns of the one-parameter Case 1 family)
    assert np.linalg.norm(W - Wr @ (Wr.T @ W), 2) <= 1e-4
    assert np.abs(res["ANq"][:, :2, :2] - ref["ANq"][:, :2, :2]).max() <= 1e-9 * np.abs(ref["ANq"]).max()
    assert np.abs(res["fn"][:, :2] - ref["fnr"][:, :2]).max() <= 1e-9 * np.abs(ref["fnr"]).max()
