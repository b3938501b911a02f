"""Device-resident SPG (spg.py drop-in) against the reference's own results
(tests/golden/spg.npz, written by tests/golden/make_spg_golden.py with the real
reference) and the reference's test_spg.py cases."""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "spg.npz"))


def S():
    from paper_2603_15910_b200 import spg

    return spg


def test_svm_blobs_matches_reference():
    spg = S()
    pts, labels = G["pts"], G["labels"]
    res = spg.spg_solve(spg.build_svm_dual(pts, labels, gamma=0.05, C=1.0), np.zeros(80), tol=1e-4)
    assert res.converged and bool(G["svm_conv"])
    assert abs(res.iterations - int(G["svm_it"])) <= 2
    assert abs(float(labels @ res.x)) <= 1e-8  # dual feasibility
    assert np.all(res.x >= -1e-10) and np.all(res.x <= 1.0 + 1e-10)
    np.testing.assert_allclose(res.x, G["svm_x"], atol=1e-5)
    assert abs(res.objectives[-1] - float(G["svm_obj"])) <= 1e-8 * max(1.0, abs(float(G["svm_obj"])))


@pytest.mark.parametrize("warm", [False, True])
def test_basis_pursuit_matches_reference(warm):
    spg = S()
    tag = "bp_warm" if warm else "bp_cold"
    res = spg.spg_solve(spg.build_basis_pursuit(G["A"], G["b"], radius=float(G["radius"]),
                                                warm_start=warm),
                        np.zeros(1000), tol=1e-4, max_iter=5000)
    assert res.converged and res.pg_norms[-1] < 1e-4
    ref_obj = float(G[tag + "_obj"])
    # the nonmonotone path is rounding-sensitive over hundreds of steps and
    # stops at a projected-gradient norm of 1e-4: the objective must agree
    # tightly, the iterate to the stopping tolerance, the step count closely
    assert abs(res.objectives[-1] - ref_obj) <= 1e-6 * max(1.0, abs(ref_obj))
    np.testing.assert_allclose(res.x, G[tag + "_x"], atol=1e-3)
    assert abs(res.iterations - int(G[tag + "_it"])) <= 0.1 * int(G[tag + "_it"])
    assert np.abs(res.x).sum() <= float(G["radius"]) * (1 + 1e-12)


def test_warm_starts_do_not_cost_more():
    spg = S()
    runs = {}
    for warm in (False, True):
        res = spg.spg_solve(spg.build_basis_pursuit(G["A"], G["b"], radius=float(G["radius"]),
                                                    warm_start=warm),
                            np.zeros(1000), tol=1e-4, max_iter=5000)
        runs[warm] = np.mean([c for c, _ in res.inner_iterations[-100:]])
    assert runs[True] <= runs[False] + 1e-12  # test_acceptance.py:219-238


def test_reference_unit_cases():
    spg = S()
    import paper_2603_15910_b200 as P

    pts = np.array([[0.0, 0.0], [10.0, 0.0]])
    res = spg.spg_solve(spg.build_svm_dual(pts, np.array([1.0, -1.0]), gamma=100.0, C=1.0),
                        np.zeros(2), tol=1e-8)
    np.testing.assert_allclose(res.x, [1.0, 1.0], atol=1e-6)
    b = np.array([2.0, -1.0])
    res = spg.spg_solve(spg.build_basis_pursuit(np.eye(2), b, radius=1.0), np.zeros(2), tol=1e-10)
    np.testing.assert_allclose(res.x, O.project_l1(b, 1.0)["x"], atol=1e-6)
    b = np.array([0.3, -0.2])
    res = spg.spg_solve(spg.build_basis_pursuit(np.eye(2), b, radius=1.0), np.zeros(2), tol=1e-10)
    np.testing.assert_allclose(res.x, b, atol=1e-8)
    res = spg.spg_solve(spg.build_basis_pursuit(np.eye(3), np.zeros(3), radius=1.0), np.zeros(3),
                        tol=1e-8)
    assert res.converged and res.iterations <= 1
    with pytest.raises(P.DomainError):
        spg.build_svm_dual(np.ones((4, 2)), np.ones(4), gamma=1.0, C=1.0)


def test_simplex_warm_start_matches_oracle():
    import paper_2603_15910_b200 as P

    rng = np.random.default_rng(11)
    for n in (5, 300, 5000):
        y = rng.normal(0, 1, n)
        xbar = np.maximum(0.0, rng.normal(0, 1, n))
        out = P.newton_project_simplex(y, 1.0, xbar=xbar, sharpened=True)
        ref = O.newton_project_simplex(y, 1.0, xbar=xbar, sharpened=True)
        assert abs(out.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))
        assert np.abs(out.x - ref["x"]).max() <= 1e-12
        assert out.iterations == ref["iterations"]
