"""Oracle pins for the general affine (face-coefficient) operator and the paper's
Case 1 / Case 2 problems (NEXT(4), DESIGN.md AMB-23; Table 1)."""
import numpy as np
import pytest

import refs
from synth import cases

RNG = np.random.default_rng(23)


@pytest.mark.parametrize("dim,m,blocks", [(2, 7, (3, 3)), (2, 10, (2, 3)), (3, 5, (2, 2, 2))])
def test_faces_from_blocks_is_the_block_operator(orc, dim, m, blocks):
    """The face operator with the cell-average faces of the thermal blocks equals the
    block operator (AMB-1) -- apply, Gauss-Seidel, Jacobi and an RBCG solve."""
    gb = orc.Grid(dim, m, blocks)
    gf = orc.Grid(dim, m, faces=cases.faces_from_blocks(dim, m, blocks))
    assert gf.Q == gb.Q
    th = 0.1 * 100 ** RNG.random(gb.Q)
    x = RNG.standard_normal(gb.N)
    b = RNG.standard_normal(gb.N)
    ya, yb = gb.apply_A(th, x), gf.apply_A(th, x)
    assert np.abs(ya - yb).max() <= 1e-14 * np.abs(ya).max()
    for c in (0, 1):
        ga, gbb = gb.gs_halfsweep(th, b, x, c), gf.gs_halfsweep(th, b, x, c)
        assert np.abs(ga - gbb).max() <= 1e-14 * np.abs(ga).max()
    ja, jb = gb.smooth(th, b, x, orc.JACOBI, 2, 0.8), gf.smooth(th, b, x, orc.JACOBI, 2, 0.8)
    assert np.abs(ja - jb).max() <= 1e-14 * np.abs(ja).max()
    ra, rb = gb.rbcg(None, None, None, th, b=b), gf.rbcg(None, None, None, th, b=b)
    assert ra["status"] == rb["status"] == "CONVERGED" and abs(ra["its"] - rb["its"]) <= 1
    assert np.linalg.norm(ra["x"] - rb["x"]) <= 1e-9 * np.linalg.norm(ra["x"])


def test_face_operator_matches_independent_fd_assembly(orc):
    """faces_from_blocks + the oracle's face operator == the cell-wise FD assembly of tests/refs.py."""
    dim, m, blocks = 3, 4, (2, 2, 2)
    gf = orc.Grid(dim, m, faces=cases.faces_from_blocks(dim, m, blocks))
    th = 0.1 * 100 ** RNG.random(gf.Q)
    A = refs.cellwise_fd(dim, m, blocks, th).toarray()
    assert np.abs(gf.dense_A(th) - A).max() <= 1e-12 * np.abs(A).max()


@pytest.mark.parametrize("case", [1, 2])
def test_case_operators_spd_and_affine(orc, case):
    m = 5
    P = cases.case_problem(case, m)
    g = orc.Grid(3, m, faces=P["faces"])
    mu = cases.case_params(case, 1, 3)[0]
    th = P["theta"](mu)
    A = g.dense_A(th)
    assert np.abs(A - A.T).max() <= 1e-12 * np.abs(A).max()
    assert np.linalg.eigvalsh(A).min() > 0
    # affine: A(theta) = A_0 + mu_1 A_1 with A_q the single-field operators
    A0 = g.dense_A(np.array([1.0, 0.0]))
    A1 = g.dense_A(np.array([0.0, 1.0]))
    assert np.abs(A - (A0 + mu[0] * A1)).max() <= 1e-12 * np.abs(A).max()


def test_case1_manufactured_solution_second_order(orc):
    """Case 1 at mu = 0 is -Laplace u = 3 pi^2 sin sin sin: u = sin(pi x) sin(pi y) sin(pi z);
    the discrete solution's max error falls by ~4 per halving of h."""
    errs = []
    for m in (7, 15):
        P = cases.case_problem(1, m)
        g = orc.Grid(3, m, faces=P["faces"])
        f = P["terms"][0]
        r = g.rbcg(None, None, None, P["theta"](np.array([0.0])), b=f, tol=1e-12)
        assert r["status"] == "CONVERGED"
        x, y, z = cases.node_xyz(3, m)
        u = np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)
        errs.append(np.abs(r["x"] - u).max())
    assert 3.5 <= errs[0] / errs[1] <= 4.5, errs


def test_dirichlet_lifting_reproduces_a_linear_profile(orc):
    """With kappa = 1 (mu_1 = 0) and no source, boundary data g linear in x, y, z gives the
    discrete solution g at the interior nodes (the 7-point scheme is exact on linear
    functions): pins the lifting terms of Case 2."""
    m = 6
    F = cases.faces_from_nodal(3, m, cases.kappa_fields(2))
    g = orc.Grid(3, m, faces=F)

    def lin(x, y, z):
        return 0.3 + x + 2 * y - 1.5 * z

    L = cases.lifting(3, m, F, lin)
    th = np.array([1.0, 0.0])
    b = th[0] * L[0] + th[1] * L[1]
    r = g.rbcg(None, None, None, th, b=b, tol=1e-13)
    x, y, z = cases.node_xyz(3, m)
    assert np.abs(r["x"] - lin(x, y, z)).max() <= 1e-10


def test_case2_rhs_terms_are_the_bilinear_expansion(orc):
    """f(mu) = sum_r phi_r(mu) t_r equals source + lifting of (1 + mu1 F1)((1-mu2) g_a + mu2 g_b)
    assembled directly with the blended faces and profile."""
    m = 5
    P = cases.case_problem(2, m)
    mu = np.array([1.3, 0.4])
    rhs = P["phi"](mu) @ P["terms"]
    Fb = (P["faces"][0] + mu[0] * P["faces"][1])[None]

    def g(x, y, z):
        ga = np.cos(10 * np.pi * (4 * (x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2))
        gb = np.cos(10 * np.pi * (x + y + z))
        return (1 - mu[1]) * ga + mu[1] * gb

    direct = cases.source(3, m) + cases.lifting(3, m, Fb, g)[0]
    assert np.abs(rhs - direct).max() <= 1e-12 * np.abs(direct).max()
    assert np.allclose(P["phi"](np.array([1.0, 0.5])), [1, 0.5, 0.5, 0.5, 0.5])


def test_affine_rhs_greedy_reduces_to_the_constant_rhs(orc):
    """or_set_greedy_rhs with one term f_1 = 1, phi = 1 is the f = 1 greedy (same snapshots,
    selections, basis); its f_{N,1} equals the offline fn = W^T 1."""
    g = orc.Grid(2, 15, (2, 2))
    rng = np.random.default_rng(4)
    tr = 0.1 * 100 ** rng.random((12, g.Q))
    a = g.greedy(tr, 4)
    b = g.greedy(tr, 4, phi_train=np.ones((12, 1)), terms=np.ones((1, g.N)))
    assert np.array_equal(a["selected"], b["selected"])
    assert np.abs(a["W"] - b["W"]).max() <= 1e-13
    assert np.abs(b["fnr"][0] - a["fn"]).max() <= 1e-12 * np.abs(a["fn"]).max()
