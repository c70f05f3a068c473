"""The §8(b) boundary calls added in round 2 (include/rbs.h), against the oracle:
affine right-hand-side terms with the online f_N(mu) = sum_r phi_r f_{N,r} (PAPER.md:
105-115 eq12b), the parameter map, the cell-label operator, and the query-sharding
communicator + basis broadcast (a one-rank communicator: the boxes have one GPU)."""
import numpy as np
import pytest

from test_gpu_parity import compare, rbs  # noqa: F401  (fixture)
from synth import cases

pytestmark = pytest.mark.gpu


def _affine_problem(orc, seed=5):
    """2D 31^2, 2x2 blocks, R = 3 random right-hand-side terms, greedy basis built by the
    oracle with the affine right-hand side (or_set_greedy_rhs)."""
    g = orc.Grid(2, 31, (2, 2))
    rng = np.random.default_rng(seed)
    terms = rng.standard_normal((3, g.N)) + 1.0
    tr = 0.1 * 100 ** rng.random((30, 4))
    phi_tr = rng.random((30, 3)) + 0.5
    res = g.greedy(tr, 8, phi_train=phi_tr, terms=terms)
    return g, terms, res


@pytest.mark.parametrize("method", ["rbcg", "rbi"])
def test_rhs_terms_online_match_oracle(orc, rbs, method):
    """theta = mu (identity map), phi from an affine map of 4 parameters: the solve forms
    f(mu) on the device and f_N(mu) from the offline f_{N,r} (no rhs_dev); results match
    the oracle solving with b = sum_r phi_r f_r, and the explicit-rhs path of the library."""
    import torch
    g, terms, res = _affine_problem(orc)
    rng = np.random.default_rng(9)
    Pa = np.hstack([rng.random((3, 1)) + 0.2, 0.1 * rng.random((3, 4))])     # phi = Pa [1; mu]
    s = rbs.Solver(2, 31, (2, 2)).set_rhs_terms(terms).set_param_map(4, None, Pa)
    s.load_basis(res["W"], res["ANq"], res["fn"])
    # offline f_{N,r} = W^T f_r computed by the library equals the oracle greedy's
    mus = 0.1 * 100 ** rng.random((5, 4))
    phi = np.stack([Pa @ np.concatenate([[1.0], mu]) for mu in mus])
    kw = dict(method=rbs.RBS_RBCG if method == "rbcg" else rbs.RBS_RBI,
              max_iter=20000 if method == "rbcg" else 500000, record_history=1)
    out = s.solve_batch(mus, **kw)
    for b in range(len(mus)):
        f = phi[b] @ terms
        solve = g.rbcg if method == "rbcg" else g.rbi
        ref = solve(res["W"], res["ANq"], res["fn"], mus[b], b=f, max_iter=kw["max_iter"])
        assert out["status"][b] == ref["status"] == "CONVERGED"
        assert abs(int(out["its"][b]) - ref["its"]) <= 1
        x = out["X"][b].cpu().numpy()
        assert np.linalg.norm(x - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])
        assert np.abs(out["a_n"][b] - ref["a_n"]).max() <= 1e-10 * np.abs(ref["a_n"]).max()
        k = min(len(out["history"][b]), len(ref["hist"]))
        assert np.all(np.abs(out["history"][b][:k] - ref["hist"][:k]) <= 1e-6 * ref["hist"][:k] + 1e-13)
    # the same queries with explicit right-hand sides (rhs_dev) through a plain context
    s2 = rbs.Solver(2, 31, (2, 2)).load_basis(res["W"], res["ANq"], res["fn"])
    out2 = s2.solve_batch(mus, rhs=torch.tensor(phi @ terms, device="cuda"), **kw)
    assert np.array_equal(out["its"], out2["its"])
    X1, X2 = out["X"].cpu().numpy(), out2["X"].cpu().numpy()
    assert np.linalg.norm(X1 - X2) <= 1e-11 * np.linalg.norm(X2)


def test_param_map_case2(orc, rbs):
    """The paper's Case 2 (Table 1; AMB-23) at 15^3 with the bilinear phi written
    affinely in the derived parameters mu' = (mu_1, mu_2, mu_1 mu_2): theta = (1, mu_1),
    phi = (1, 1 - mu_2, mu_2, mu_1 - mu_1 mu_2, mu_1 mu_2)."""
    m = 15
    P = cases.case_problem(2, m)
    g = orc.Grid(3, m, faces=P["faces"])
    tr = cases.case_params(2, 24, 1002)
    res = g.greedy(np.stack([P["theta"](mu) for mu in tr]), 6,
                   phi_train=np.stack([P["phi"](mu) for mu in tr]), terms=P["terms"])
    Ta = np.array([[1.0, 0, 0, 0], [0, 1.0, 0, 0]])
    Pa = np.array([[1.0, 0, 0, 0], [1.0, 0, -1.0, 0], [0, 0, 1.0, 0], [0, 1.0, 0, -1.0], [0, 0, 0, 1.0]])
    s = rbs.Solver(3, m, faces=P["faces"]).set_rhs_terms(P["terms"]).set_param_map(3, Ta, Pa)
    s.load_basis(res["W"], res["ANq"], res["fnr"][0])
    q = cases.case_params(2, 6, 2002)
    mup = np.stack([[a, b_, a * b_] for a, b_ in q])
    out = s.solve_batch(mup, record_history=1)
    for b, mu in enumerate(q):
        ref = g.rbcg(res["W"], res["ANq"], res["fnr"][0], P["theta"](mu), b=P["phi"](mu) @ P["terms"])
        assert out["status"][b] == ref["status"] and abs(int(out["its"][b]) - ref["its"]) <= 1
        x = out["X"][b].cpu().numpy()
        assert np.linalg.norm(x - ref["x"]) <= 1e-9 * np.linalg.norm(ref["x"])


@pytest.mark.parametrize("dim,m,blocks", [(2, 37, (3, 3)), (3, 13, (2, 2, 2))])
def test_labels_operator_equals_blocks(orc, rbs, dim, m, blocks):
    """Cell labels from the thermal-block partition (AMB-2: block of the cell centre) give
    the block operator: the label context matches the oracle's block operator."""
    p = list(blocks) + [1] * (3 - len(blocks))
    a = np.arange(m + 1)
    bl = [((2 * a + 1) * p[k]) // (2 * (m + 1)) for k in range(3)]
    if dim == 2:
        lab = bl[0][None, :] + p[0] * bl[1][:, None]                 # [b][a], x fastest
    else:
        lab = (bl[0][None, None, :] + p[0] * bl[1][None, :, None] + p[0] * p[1] * bl[2][:, None, None])
    g = orc.Grid(dim, m, blocks)
    tr = 0.1 * 100 ** np.random.default_rng(4).random((30, g.Q))
    res = g.greedy(tr, 6)
    s = rbs.Solver(dim, m, blocks).set_labels(lab.reshape(-1).astype(np.uint8))
    s.load_basis(res["W"], res["ANq"], res["fn"])
    mus = 0.1 * 100 ** np.random.default_rng(5).random((4, g.Q))
    out = s.solve_batch(mus, record_history=1)
    compare(out, g, res["W"], res["ANq"], res["fn"], mus, "rbcg")
    A, f = rbs.Solver(dim, m, blocks).set_labels(lab.reshape(-1).astype(np.uint8)).load_basis(res["W"]).offline_blocks()
    assert np.abs(A - res["ANq"]).max() <= 1e-12 * np.abs(res["ANq"]).max()


def test_comm_broadcast_single_rank(orc, rbs):
    """rbs_comm_init + rbs_broadcast_basis on a one-rank NCCL communicator (root = this
    rank): the collective runs (graph of a broadcast of the storage prefix), the solve
    after it is bitwise the solve before it; the argument checks fire."""
    g = orc.Grid(2, 31, (2, 2))
    tr = 0.1 * 100 ** np.random.default_rng(6).random((30, 4))
    res = g.greedy(tr, 6)
    s = rbs.Solver(2, 31, (2, 2)).load_basis(res["W"], res["ANq"], res["fn"])
    mus = tr[:3]
    a = s.solve_batch(mus)
    with pytest.raises(rbs.RbsError, match="E_STATE"):
        s.broadcast_basis(0, res["n"])                 # no communicator yet
    s.comm_init(rbs.rbs_nccl_unique_id(), 1, 0)
    with pytest.raises(rbs.RbsError, match="E_STATE"):
        rbs.rbs_broadcast_basis(s.ctx, 0, res["n"] + 1, s._storage)   # root without that n
    s.broadcast_basis(0, res["n"])
    b = s.solve_batch(mus)
    assert np.array_equal(a["X"].cpu().numpy(), b["X"].cpu().numpy())
