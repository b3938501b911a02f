"""Algorithm 2 on the device (simplex.py:47-154) and its chunked form
(parallel.py:330-368) against the REAL reference's fixtures and the oracle:
bit-exact multipliers, free sets and zero proofs; then the Algorithm-2
Newton route of newton_project_simplex / project_l1."""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_simplex_init_lambda_bitexact_vs_reference_fixtures():
    import paper_2603_15910_b200 as P

    z = np.load(os.path.join(G, "small.npz"))
    for k in range(int(z["n_spx"][0])):
        p = f"s{k}_"
        y, r = z[p + "y"], float(z[p + "r"][0])
        init = P.simplex_init_lambda(y, r)
        assert init.lambda0 == z[p + "init_lam"][0], k
        assert np.array_equal(np.asarray(init.free), z[p + "init_free"]), k


def test_simplex_init_lambda_options_vs_oracle():
    import paper_2603_15910_b200 as P

    rng = np.random.default_rng(3)
    for _ in range(60):
        n = int(rng.integers(1, 400))
        y = rng.normal(0, 1, n)
        r = float(rng.uniform(0.1, 3))
        xb = np.abs(rng.normal(0, 1, n)) * (rng.uniform(0, 1, n) > 0.5)
        for sharp in (False, True):
            yy = np.abs(y) if sharp else y
            a = P.simplex_init_lambda(yy, r, xbar=xb, sharpened=sharp)
            lam, free, fixed, sj = O.simplex_init_lambda(yy, r, xbar=xb, sharpened=sharp)
            assert a.lambda0 == lam and np.array_equal(a.free, free)
            assert np.array_equal(a.fixed_mask, fixed)
    with pytest.raises(P.EmptyIndexSet):
        P.simplex_init_lambda(np.ones(3), 1.0, idx=np.array([], np.int64))


@pytest.mark.parametrize("workers", [1, 2, 3, 7, 64, 1000])
def test_par_simplex_init_bitexact_vs_oracle(workers):
    import paper_2603_15910_b200 as P

    rng = np.random.default_rng(workers)
    for _ in range(10):
        n = int(rng.integers(workers, 20000))
        y = rng.normal(0, 1, n)
        r = float(rng.uniform(0.1, 3))
        a = P.par_simplex_init(y, r, workers=workers)
        lam, free, fixed, sj = O.par_simplex_init(y, r, workers)
        assert a.lambda0 == lam and a.sum_free == sj
        assert np.array_equal(a.free, free) and np.array_equal(a.fixed_mask, fixed)


@pytest.mark.parametrize("family", ["simplex-u01", "simplex-n01", "simplex-n0m3"])
def test_alg2_route_matches_reference(family):
    import paper_2603_15910_b200 as P

    for n in (1000, 100_000, 1_000_000):
        y = P.gen_simplex_y(family, n, 1)
        o = P.newton_project_simplex(y, 1.0, start="alg2")
        lam_star = O.exact_simplex_lambda(y, 1.0)
        ref = O.newton_project_simplex(y, 1.0)  # the reference's default (Algorithm 2) route
        assert abs(o.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))
        assert abs(o.lam - lam_star) <= 1e-12 * max(1.0, abs(lam_star))
        assert float(np.abs(o.x - ref["x"]).max()) <= 1e-12
        # replay: the same chunked init + Algorithm 4 in the oracle
        W = max(1, min(n // 256, P._native.handle().info()["sm_count"] * 1024))
        lam0, free, fixed, _ = O.par_simplex_init(y, 1.0, W)
        lam0 = min(lam0, 1.0 - float(y[free].max()))  # both upper bounds of the root
        rr = O.newton_simplex_from(y, 1.0, lam0, np.flatnonzero(~fixed))
        assert o.iterations == rr["iterations"] and o.fixed_count == rr["fixed_count"]
        assert abs(o.lam - rr["lam"]) <= 1e-12 * max(1.0, abs(rr["lam"]))


def test_alg2_route_l1():
    import paper_2603_15910_b200 as P

    rng = np.random.default_rng(9)
    for n in (10, 1000, 300_000):
        y = rng.normal(0, 1, n)
        for r in (0.5, 5.0, 1e9):
            x = P.project_l1(y, r, start="alg2")
            ref = O.project_l1(y, r)
            assert float(np.abs(x - ref["x"]).max()) <= 1e-12, (n, r)
