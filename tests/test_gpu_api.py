"""Drop-in API details the reference's callers rely on: the sharpened
simplex route (simplex.py:243-245; the answer changes when lambda* > 0), the
l1 warm start's xbar check after the inside-the-ball test (simplex.py:
311-333, 139-140), the top-level SPG names (__init__.py:37), and float32
instances (test_newton.py:212-220, test_simplex.py:224-228)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def test_sharpened_simplex_with_positive_root():
    import paper_2603_15910_b200 as P

    rng = np.random.default_rng(5)
    for n in (3, 50, 5000, 200_000):
        y = rng.normal(0.0, 1.0, n)
        r = float(np.abs(y).sum()) + 3.0  # the root is positive
        for sharp in (False, True):
            ref = O.newton_project_simplex(y, r, sharpened=sharp)
            out = P.newton_project_simplex(y, r, sharpened=sharp)
            assert abs(out.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"])), (n, sharp)
            assert np.abs(out.x - ref["x"]).max() <= 1e-12 * max(1.0, r)
        # the two routes really differ here: sharpened keeps every y_i <= 0 out
        # of the multiplier updates (simplex.py:79-80), so the root moves; the
        # dense x is still max(0, y + lam) everywhere (simplex.py:298)
        a = P.newton_project_simplex(y, r, sharpened=False)
        b = P.newton_project_simplex(y, r, sharpened=True)
        if (y <= 0).any():
            assert a.lam != b.lam
        assert np.array_equal(b.x, np.maximum(0.0, y + b.lam))


def test_l1_negative_xbar():
    import paper_2603_15910_b200 as P

    y = np.array([0.5, -2.0, 1.0, 0.25])
    bad = np.array([0.1, -0.3, 0.2, 0.0])
    with pytest.raises(P.DomainError) as e:
        P.project_l1(y, 1.0, xbar=bad)
    assert e.value.field == "xbar"
    inside = P.project_l1(y * 0.1, 1.0, xbar=bad)  # inside the ball: returned unchanged
    assert np.array_equal(inside, y * 0.1)
    good = np.abs(P.project_l1(y, 1.0))
    x = P.project_l1(y, 1.0, xbar=good)
    ref = O.project_l1(y, 1.0)
    assert np.abs(x - ref["x"]).max() <= 1e-12


def test_spg_names_at_top_level():
    import paper_2603_15910_b200 as P

    for name in ("SpgProblem", "SpgResult", "spg_solve", "build_svm_dual", "build_basis_pursuit",
                 "gen_blobs", "gen_sparse_ls", "par_simplex_init"):
        assert hasattr(P, name), name
    pts, labels = P.gen_blobs(40, 3, 3.0, 1)
    prob = P.build_svm_dual(pts, labels, gamma=0.5, C=10.0)
    res = P.spg_solve(prob, np.zeros(40), tol=1e-6, max_iter=500)
    assert res.converged


@pytest.mark.parametrize("kind", ["cqk", "simplex", "l1"])
def test_float32_instances(kind):
    """float32 in, float32 out on the float32 path (element math in float32,
    fp64 sums, tau = eps32^(3/4), newton.py:64-67): the multiplier agrees with
    the oracle's fp64 root to the float32 tolerance and x to float32 rounding
    (parity with the reference's own float32 runs: test_gpu_f32.py)."""
    import paper_2603_15910_b200 as P

    rng = np.random.default_rng(11)
    n = 100_000
    tau32 = float(np.finfo(np.float32).eps) ** 0.75
    if kind == "cqk":
        d, a, b, l, u, r = O.gen_cqk("cqk-weakly-correlated", n, 3)
        inst = P.CqkInstance(*[v.astype(np.float32) for v in (d, a, b, l, u)], r=r)
        out = P.solve_cqk(inst)
        ref = O.solve_cqk(*[v.astype(np.float32).astype(np.float64) for v in (d, a, b, l, u)], r)
        assert out.x.dtype == np.float32
        assert abs(out.lam - ref["lam"]) <= 10 * tau32 * max(1.0, abs(ref["lam"]))
        assert np.abs(out.x - ref["x"]).max() <= 1e-4 * max(1.0, np.abs(ref["x"]).max())
    else:
        y = rng.normal(0.0, 1.0, n).astype(np.float32)
        y64 = y.astype(np.float64)
        if kind == "simplex":
            out = P.newton_project_simplex(y, 1.0)
            ref = O.newton_project_simplex(y64, 1.0)
            x = out.x
        else:
            x = P.project_l1(y, 1.0)
            ref = O.project_l1(y64, 1.0)
        assert x.dtype == np.float32
        assert np.abs(x - ref["x"]).max() <= 1e-6
        assert abs(float(np.abs(x.astype(np.float64)).sum()) - 1.0) <= 1e-5
