"""GPU parity: the sm_100a solver vs the C oracle on identical inputs.

Bars: lambda within 1e-12 * max(1, |lambda|), x within
1e-12 * max(1, |x|_inf), identical status / iteration counts / fixed counts,
feasibility |b'x - r| <= max(1e-12 sum|b x|, tau (sum|b x| + |r|)).
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-12


def P():
    import paper_2603_15910_b200 as p

    return p


def box(d, a, b, l, u, r):
    p = P()
    return p.CqkInstance(d=np.array(d, float), a=np.array(a, float), b=np.array(b, float),
                         l=np.array(l, float), u=np.array(u, float), r=r)


def random_arrays(seed, n):
    # the reference's tests/test_core.py random_instance recipe
    rng = np.random.default_rng(seed)
    d = rng.uniform(0.5, 3.0, n)
    a = rng.normal(0.0, 2.0, n)
    b = rng.uniform(0.5, 3.0, n)
    lo = rng.normal(0.0, 1.0, n)
    hi = lo + rng.uniform(0.0, 2.0, n)
    r = float(b @ lo + rng.uniform(0, 1) * (b @ hi - b @ lo))
    return d, a, b, lo, hi, r


def close(x, y, tol=TOL):
    return abs(x - y) <= tol * max(1.0, abs(y))


def check_against(out, ref, inst_arrays, n_check_x=True):
    p = P()
    if ref["status"] == O.INFEASIBLE:
        assert out.status is p.Status.INFEASIBLE
        assert out.lam is None and out.x is None
        return
    assert ref["status"] == O.SOLVED
    assert out.status is p.Status.SOLVED
    assert close(out.lam, ref["lam"]), (out.lam, ref["lam"])
    assert out.iterations == ref["iterations"]
    assert out.phi_evals == ref["phi_evals"]
    assert out.fixed_count == ref["fixed_count"]
    if n_check_x:
        xs = max(1.0, float(np.abs(ref["x"]).max()))
        assert float(np.abs(out.x - ref["x"]).max()) <= TOL * xs


@pytest.mark.parametrize("fix", [True, False])
def test_random_instances_solve(fix):
    p = P()
    for seed in range(120):
        d, a, b, l, u, r = random_arrays(seed, 1 + seed % 60)
        inst = p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
        out = p.solve_cqk(inst, p.SolverOptions(variable_fixing=fix))
        ref = O.solve_cqk(d, a, b, l, u, r, fixing=fix)
        check_against(out, ref, (d, a, b, l, u))


def test_random_instances_jacobi_and_par():
    p = P()
    for seed in range(60):
        d, a, b, l, u, r = random_arrays(seed + 500, 50 + 37 * seed)
        inst = p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
        out = p.jacobi_solve(inst)
        ref = O.jacobi_solve(d, a, b, l, u, r, workers=1)
        check_against(out, ref, (d, a, b, l, u))
        assert out.fixed_count == 0
        out = p.par_solve_cqk(inst, workers=4)
        ref = O.par_solve_cqk(d, a, b, l, u, r, workers=4)
        assert out.status.value == ("solved" if ref["status"] == 0 else "infeasible")
        if ref["status"] == 0:
            assert close(out.lam, ref["lam"])
            assert out.fixed_count == ref["fixed_count"]


def test_hand_goldens():
    p = P()
    out = p.solve_cqk(box([1, 2], [0, 0], [1, 1], [0, 0], [1, 1], 1.0))
    assert out.status is p.Status.SOLVED
    assert abs(out.lam - 2 / 3) <= 1e-14
    np.testing.assert_allclose(out.x, [2 / 3, 1 / 3], atol=1e-14)
    out = p.solve_cqk(box([1, 1], [0, 0], [1, 1], [0, 0], [0, 0], 1.0))
    assert out.status is p.Status.INFEASIBLE and out.lam is None and out.x is None
    inst = box([2, 3], [1, -1], [1, 2], [0, 0], [1, 1], 3.0)
    out = p.solve_cqk(inst)
    np.testing.assert_allclose(out.x, inst.u, atol=1e-12)
    out = p.solve_cqk(box([2.0], [1.0], [3.0], [0.0], [5.0], 6.0))
    assert abs(out.x[0] - 2.0) <= 1e-12
    for solver in (p.jacobi_solve, p.par_solve_cqk):
        out = solver(box([1, 1], [0, 0], [1, 1], [0, 0], [0, 0], 1.0))
        assert out.status is p.Status.INFEASIBLE


def test_domain_errors():
    p = P()
    with pytest.raises(p.DomainError) as e:
        p.solve_cqk(box([1, -1], [0, 0], [1, 1], [0, 0], [1, 1], 1.0))
    assert e.value.field == "d" and e.value.index == 1
    with pytest.raises(p.DomainError) as e:
        p.validate(box([1], [0], [1], [2], [1], 1.0))
    assert e.value.field == "bounds" and e.value.index == 0
    with pytest.raises(p.DomainError):
        p.validate(box([1], [0], [0], [0], [1], 1.0))
    with pytest.raises(p.DomainError) as e:
        p.validate(box([1], [0], [1], [0], [1], np.inf))
    assert e.value.field == "r"
    with pytest.raises(p.DomainError) as e:
        p.validate(box([1, 1, 1], [0, np.nan, 0], [1, 1, 1], [0, 0, 0], [1, 1, 1], 1.0))
    assert e.value.field == "a" and e.value.index == 1


def test_eval_phi_goldens():
    p = P()
    inst = p.simplex_as_cqk(np.array([1.0, 2.0, 3.0]), 1.0)
    ph = p.eval_phi(inst, -2.0)
    assert ph.value == 1.0 and ph.dplus == 2.0 and ph.dminus == 1.0
    two = box([1, 2], [0, 0], [1, 1], [0, 0], [1, 1], 1.0)
    ph = p.eval_phi(two, -10.0)
    assert ph.value == 0.0 and ph.dplus == 0.0 and ph.dminus == 0.0
    ph = p.eval_phi(two, 2 / 3)
    assert abs(ph.value - 1.0) <= 1e-15 and ph.dplus == 1.5 and ph.dminus == 1.5
    ph = p.eval_phi(box([1, 1], [0, 0], [1, 1], [0, 0], [0, 0], 0.0), 0.0)
    assert ph.value == 0.0 and ph.dplus == 0.0 and ph.dminus == 0.0
    np.testing.assert_allclose(p.eval_x(two, 2 / 3), [2 / 3, 1 / 3])
    assert np.array_equal(p.eval_x(two, 100.0), two.u)
    assert p.eval_x(two, 0.4, np.array([1]))[0] == p.eval_x(two, 0.4)[1]


def test_phi_scan_matches_oracle_bitwise_on_masks():
    p = P()
    for seed in range(30):
        d, a, b, l, u, r = random_arrays(seed + 900, 300)
        inst = p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
        for lam in (-3.0, -0.5, 0.0, 0.7, 2.5):
            idx = np.arange(0, 300, 3)
            got = p.core.phi_scan(inst, lam, idx, masks=True)
            ref = O.phi_scan(d, a, b, l, u, lam, idx)
            for k in range(4):
                assert abs(got[k] - ref[k]) <= 1e-13 * max(1.0, abs(ref[k]))
            assert np.array_equal(got[4], ref[4]) and np.array_equal(got[5], ref[5])


def test_nearest_breakpoint_goldens():
    p = P()
    from paper_2603_15910_b200.newton import Direction

    inst = p.simplex_as_cqk(np.array([0.0, -1.0, -2.0]), 1.0)
    st = p.SolveState(active=np.arange(3), r_residual=1.0, bracket_lo=0.5)
    assert p.nearest_breakpoint(st, inst, Direction.RIGHT) == 1.0
    st = p.SolveState(active=np.arange(3), r_residual=1.0, bracket_hi=0.0)
    assert p.nearest_breakpoint(st, inst, Direction.LEFT) is None
    inst = p.simplex_as_cqk(np.array([0.0, 0.0, -3.0]), 1.0)
    st = p.SolveState(active=np.arange(3), r_residual=1.0, bracket_lo=0.0)
    assert p.nearest_breakpoint(st, inst, Direction.RIGHT) == 3.0


def test_initial_multiplier():
    p = P()
    inst = p.simplex_as_cqk(np.array([1.0, 2.0, 3.0]), 1.0)
    assert abs(p.initial_multiplier(inst) + 5 / 3) <= 1e-15
    two = box([1, 2], [0, 0], [1, 1], [0, 0], [1, 1], 1.0)
    assert p.initial_multiplier(two, xbar=np.array([0.0, 1.0])) == p.initial_multiplier(two)
    assert abs(p.initial_multiplier(two, xbar=np.array([0.5, 1.0])) - 1.0) <= 1e-15


def test_bit_identical_reruns():
    p = P()
    d, a, b, l, u, r = p.instances.gen_cqk_arrays("cqk-weakly-correlated", 300000, 3)
    inst = p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
    o1 = p.solve_cqk(inst)
    o2 = p.solve_cqk(inst)
    assert o1.lam == o2.lam and np.array_equal(o1.x, o2.x)


@pytest.mark.parametrize("family", ["cqk-uncorrelated", "cqk-weakly-correlated", "cqk-correlated"])
def test_generated_1e6(family):
    p = P()
    for seed in (1, 2):
        d, a, b, l, u, r = p.instances.gen_cqk_arrays(family, 10**6, seed)
        inst = p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
        for fix in (True, False):
            out = p.solve_cqk(inst, p.SolverOptions(variable_fixing=fix))
            ref = O.solve_cqk(d, a, b, l, u, r, fixing=fix)
            check_against(out, ref, (d, a, b, l, u))
            x = out.x
            bx = b * x
            resid = abs(float(bx.sum()) - r)
            tau = O.TAU64
            assert resid <= max(1e-12 * float(np.abs(bx).sum()), tau * (float(np.abs(bx).sum()) + abs(r)))


def test_simplex_random_vs_oracle():
    p = P()
    rng = np.random.default_rng(13)
    for _ in range(150):
        n = int(rng.integers(1, 400))
        y = rng.normal(0, 1, n)
        r = float(rng.uniform(0.1, 3))
        for start in ("formula", "tight"):
            out = p.newton_project_simplex(y, r, start=start)
            lam0 = (r - O.pairwise_sum(y)) / n
            if start == "tight":
                lam0 = min(lam0, r - float(y.max()))
            ref = O.newton_project_simplex(y, r, lam0=lam0)
            assert close(out.lam, ref["lam"]), (out.lam, ref["lam"])
            assert out.iterations == ref["iterations"], (start, out.iterations, ref["iterations"])
        auto = p.newton_project_simplex(y, r)
        assert close(auto.lam, ref["lam"]), (auto.lam, ref["lam"])
        assert float(np.abs(auto.x - ref["x"]).max()) <= TOL * max(1.0, float(np.abs(y).max()))
        assert float(np.abs(out.x - ref["x"]).max()) <= TOL * max(1.0, float(np.abs(y).max()))
        lam_star = O.exact_simplex_lambda(y, r)
        assert abs(out.lam - lam_star) <= 1e-10 * max(1.0, abs(lam_star))


def test_simplex_goldens_and_trace():
    p = P()
    out = p.newton_project_simplex(np.array([2.0, 1.0]), 1.0)
    assert abs(out.lam + 1.0) <= 1e-12
    np.testing.assert_allclose(out.x, [1.0, 0.0], atol=1e-12)
    out = p.newton_project_simplex(np.zeros(9), 9.0)
    np.testing.assert_allclose(out.x, np.ones(9), atol=1e-12)
    out = p.newton_project_simplex(np.array([2.0, 1.0]), 1.0, output="sparse")
    idx, vals = out.sparse
    assert out.x is None and list(idx) == [0]
    np.testing.assert_allclose(vals, [1.0], atol=1e-14)
    y = np.array([0.5, 0.2, 0.9])
    for lam0 in (5.0, 0.0, -0.05, -2.0):
        tr = []
        out = p.newton_project_simplex(y, 1.0, lambda0=lam0, trace=tr)
        np.testing.assert_allclose(out.x, [0.3, 0.0, 0.7], atol=1e-10)
        ref = O.newton_project_simplex(y, 1.0, lam0=lam0, trace=True)
        assert len(tr) == len(ref["trace"])
        for g, e in zip(tr, ref["trace"]):
            assert all(close(gv, ev) for gv, ev in zip(g, e))


def test_l1_random_vs_oracle():
    p = P()
    rng = np.random.default_rng(23)
    for _ in range(150):
        n = int(rng.integers(1, 300))
        y = rng.normal(0, 1, n)
        r = float(rng.uniform(0.05, 1.2) * max(0.1, np.abs(y).sum()))
        x = p.project_l1(y, r)
        ref = O.project_l1(y, r)
        if ref["iterations"] == -1:
            assert np.array_equal(x, y)
        else:
            assert float(np.abs(x - ref["x"]).max()) <= TOL * max(1.0, float(np.abs(y).max()))
            assert abs(float(np.abs(x).sum()) - r) <= 1e-10 * max(1.0, r)
    np.testing.assert_allclose(p.project_l1(np.array([2.0, -1.0]), 1.0), [1.0, 0.0], atol=1e-12)
    np.testing.assert_allclose(p.project_l1(np.array([0.0, 3.0]), 1.0), [0.0, 1.0], atol=1e-12)


def test_rows_vs_oracle():
    p = P()
    rng = np.random.default_rng(5)
    for cols in (1, 3, 255, 256, 257, 1000, 4096, 8192):
        Y = rng.normal(0, 1, (17, cols))
        X, lam, its, _ = p.project_simplex_rows(Y, 1.0)
        for i in range(Y.shape[0]):
            lam0 = min((1.0 - O.pairwise_sum(Y[i])) / cols, 1.0 - float(Y[i].max()))
            ref = O.newton_project_simplex(Y[i], 1.0, lam0=lam0)
            assert close(lam[i], ref["lam"]), (cols, i, lam[i], ref["lam"])
            assert its[i] == ref["iterations"]
            assert float(np.abs(X[i] - ref["x"]).max()) <= TOL * max(1.0, float(np.abs(Y[i]).max()))


def test_device_tensors_zero_copy():
    import torch

    p = P()
    d, a, b, l, u, r = p.instances.gen_cqk_arrays("cqk-correlated", 100000, 4)
    dev = [torch.from_numpy(v).cuda() for v in (d, a, b, l, u)]
    inst = p.CqkInstance(*dev, r=r)
    out = p.solve_cqk(inst)
    ref = O.solve_cqk(d, a, b, l, u, r)
    assert out.x.is_cuda
    assert close(out.lam, ref["lam"])
    assert float((out.x.cpu().numpy() - ref["x"]).__abs__().max()) <= 1e-12 * 25


def test_solve_pipeline_matches_sequential():
    p = P()
    from paper_2603_15910_b200.pipeline import SolvePipeline

    insts = []
    for seed in range(6):
        d, a, b, l, u, r = random_arrays(900 + seed, 5000 + 997 * seed)
        insts.append(p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r))
    seq = [p.solve_cqk(i) for i in insts]
    with SolvePipeline(depth=3) as pipe:
        outs = [f.result() for f in [pipe.submit(i) for i in insts]]
    for s, o in zip(seq, outs):
        assert o.status is s.status and o.lam == s.lam and o.iterations == s.iterations
        assert np.array_equal(o.x, s.x)


def test_rows_many_per_cta_mixed_paths():
    """More rows than resident CTAs (the next row streams in while a row
    iterates), alternating rows whose free set fits the warp buffers (zero-fill
    + scatter output) with rows that overflow them (staged output)."""
    p = P()
    rng = np.random.default_rng(9)
    rows, cols = 4001, 4096
    Y = rng.normal(0, 1, (rows, cols))
    Y[1::2] = rng.uniform(0, 1, (rows // 2, cols))  # u01 rows overflow at the tight start
    X, lam, its, _ = p.project_simplex_rows(Y, 1.0)
    for i in list(range(0, 40)) + list(range(rows - 40, rows)) + list(range(1000, 4000, 97)):
        lam0 = min((1.0 - O.pairwise_sum(Y[i])) / cols, 1.0 - float(Y[i].max()))
        ref = O.newton_project_simplex(Y[i], 1.0, lam0=lam0)
        assert close(lam[i], ref["lam"]), (i, lam[i], ref["lam"])
        assert its[i] == ref["iterations"]
        assert float(np.abs(X[i] - ref["x"]).max()) <= TOL
    np.testing.assert_allclose(X.sum(axis=1), 1.0, atol=1e-12)


@pytest.mark.parametrize("route", ["tight", "formula", "lambda0_above", "lambda0_below"])
def test_rows_start_routes_every_row(route):
    """Every start route of the batched kernel (candidate capture at max y - r,
    the second capture at lambda0, the general path) against the oracle on
    every row of a mixed batch (N(0,1) rows, u01 rows, constant rows), and
    bit-identical reruns (rows are handed out by a grid counter)."""
    p = P()
    rng = np.random.default_rng(11)
    rows, cols = 1500, 2048
    Y = rng.normal(0, 1, (rows, cols))
    Y[1::3] = rng.uniform(0, 1, (len(range(1, rows, 3)), cols))
    Y[2::15] = 0.25  # constant rows: every element ties
    kw = {}
    if route == "formula":
        kw["start"] = "formula"
    elif route == "lambda0_above":
        kw["lambda0"] = 5.0
    elif route == "lambda0_below":
        kw["lambda0"] = -5.0
    X, lam, its, _ = p.project_simplex_rows(Y, 1.0, **kw)
    X2, lam2, its2, _ = p.project_simplex_rows(Y, 1.0, **kw)
    assert np.array_equal(X, X2) and np.array_equal(lam, lam2) and np.array_equal(its, its2)
    for i in range(rows):
        y = Y[i]
        if route == "tight":
            lam0 = min((1.0 - O.pairwise_sum(y)) / cols, 1.0 - float(y.max()))
        elif route == "formula":
            lam0 = (1.0 - O.pairwise_sum(y)) / cols
        else:
            lam0 = kw["lambda0"]
        ref = O.newton_project_simplex(y, 1.0, lam0=lam0)
        assert close(lam[i], ref["lam"]), (route, i, lam[i], ref["lam"])
        assert its[i] == ref["iterations"], (route, i, its[i], ref["iterations"])
        assert float(np.abs(X[i] - ref["x"]).max()) <= TOL * max(1.0, float(np.abs(y).max()))
