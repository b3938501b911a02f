"""The two grid-step designs of the persistent TMA kernels give bit-identical
results: the single-GPU masterless step (every CTA combines the partial rows
and runs a replica of the state machine) and the master step with a release
(forced with CQK_MASTER_STEP=1; the multi-GPU path).  Both combine the rows
in the same fixed order, so lambda, the iterate counts and x must agree
bit for bit -- and both must agree with the C oracle."""
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-12


def P():
    import paper_2603_15910_b200 as p

    return p


@pytest.fixture
def tma_engine():
    from paper_2603_15910_b200 import _native as N

    h = N.handle()
    h.lib.cqk_set_engine(h.ptr, 1)
    yield
    h.lib.cqk_set_engine(h.ptr, 0)


def both_steps(fn):
    a = fn()
    b = _with_env("CQK_MASTER_STEP", fn)
    return a, b


def same(a, b):
    assert a.lam == b.lam or (np.isnan(a.lam) and np.isnan(b.lam))
    assert a.iterations == b.iterations and a.phi_evals == b.phi_evals
    assert a.fixed_count == b.fixed_count
    assert np.array_equal(a.x, b.x)


@pytest.mark.parametrize("fam", ["cqk-uncorrelated", "cqk-weakly-correlated", "cqk-correlated"])
@pytest.mark.parametrize("n", [1, 961, 300001, 2000003])
def test_cqk_master_and_masterless_agree(fam, n, tma_engine):
    p = P()
    d, a, b, l, u, r = p.instances.gen_cqk_arrays(fam, n, 3)
    inst = p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
    for opts in (p.SolverOptions(), p.SolverOptions(variable_fixing=False)):
        x, y = both_steps(lambda: p.solve_cqk(inst, opts))
        same(x, y)
    if n <= 300001:
        ref = O.solve_cqk(d, a, b, l, u, r, fixing=True)
        out = p.solve_cqk(inst)
        assert abs(out.lam - ref["lam"]) <= TOL * max(1.0, abs(ref["lam"]))
        assert out.fixed_count == ref["fixed_count"]


@pytest.mark.parametrize("fam", ["simplex-u01", "simplex-n01"])
@pytest.mark.parametrize("n", [1, 3841, 16385, 1000000])
def test_simplex_and_l1_master_and_masterless_agree(fam, n):
    p = P()
    y = p.gen_simplex_y(fam, n, 2)
    for start in ("auto", "tight", "formula"):
        x, z = both_steps(lambda: p.newton_project_simplex(y, 1.0, start=start))
        same(x, z)
        x, z = both_steps(lambda: p.simplex.project_l1_outcome(y, 1.0, start=start))
        same(x, z)


def test_masterless_repeated_launches_stay_consistent(tma_engine):
    """The arrival counters alternate between launches (each launch zeroes
    the other): many back-to-back solves of differing epoch counts."""
    p = P()
    outs = []
    for k in range(12):
        fam = ("cqk-uncorrelated", "cqk-correlated")[k % 2]
        d, a, b, l, u, r = p.instances.gen_cqk_arrays(fam, 100003 + k, k)
        inst = p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
        ref = O.solve_cqk(d, a, b, l, u, r, fixing=True)
        out = p.solve_cqk(inst)
        assert abs(out.lam - ref["lam"]) <= TOL * max(1.0, abs(ref["lam"]))
        outs.append(out.phi_evals)
    assert len(set(outs)) >= 1


@pytest.mark.parametrize("ctas", [1, 2, 37, 148])
def test_masterless_step_on_reduced_grids(ctas, tma_engine):
    """Single-GPU solves on a capped grid (cqk_set_grid_limit: a GPU shared
    with other work) run the masterless step over fewer rows."""
    from paper_2603_15910_b200 import _native as N

    p = P()
    h = N.handle()
    d, a, b, l, u, r = p.instances.gen_cqk_arrays("cqk-weakly-correlated", 200003, 5)
    inst = p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
    ref = O.solve_cqk(d, a, b, l, u, r, fixing=True)
    y = p.gen_simplex_y("simplex-u01", 100003, 5)
    lam0 = min((1.0 - float(O.pairwise_sum(y))) / y.size, 1.0 - float(y.max()))
    sref = O.newton_project_simplex(y, 1.0, lam0=lam0)
    h.lib.cqk_set_grid_limit(h.ptr, ctas)
    try:
        out = p.solve_cqk(inst)
        sp = p.newton_project_simplex(y, 1.0, start="tight")
    finally:
        h.lib.cqk_set_grid_limit(h.ptr, 0)
    assert abs(out.lam - ref["lam"]) <= TOL * max(1.0, abs(ref["lam"]))
    assert out.fixed_count == ref["fixed_count"]
    assert abs(sp.lam - sref["lam"]) <= TOL * max(1.0, abs(sref["lam"]))


def _with_env(name, fn):
    """Run fn with one of the handle's A/B switches on (cqk_set_switches;
    the environment variable of the same name sets it at handle creation)."""
    from paper_2603_15910_b200 import _native as N

    h = N.handle()
    h.set_switches(**{{"CQK_MASTER_STEP": "master_step", "CQK_STATIC_FINAL": "static_final"}[name]: True})
    try:
        return fn()
    finally:
        h.set_switches()


@pytest.mark.parametrize("n", [1, 959, 960, 961, 3841, 2000003])
def test_dynamic_and_static_final_pass_agree(n, tma_engine):
    """The final pass hands out tiles dynamically on one GPU; x is a
    per-element map, so it must equal the static walk's bit for bit."""
    p = P()
    d, a, b, l, u, r = p.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 9)
    inst = p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
    dyn = p.solve_cqk(inst)
    sta = _with_env("CQK_STATIC_FINAL", lambda: p.solve_cqk(inst))
    same(dyn, sta)
    y = p.gen_simplex_y("simplex-n01", n, 9)
    for f in (lambda: p.newton_project_simplex(y, 1.0), lambda: p.simplex.project_l1_outcome(y, 1.0)):
        same(f(), _with_env("CQK_STATIC_FINAL", f))


def test_counters_survive_interleaved_kernels(tma_engine):
    """Both persistent TMA kernels share a handle's alternating arrival and
    final-tile counters; interleave them (and the rows kernel, and static /
    master-step launches) and check every result."""
    p = P()
    y = p.gen_simplex_y("simplex-n01", 300007, 4)
    lam0 = min((1.0 - float(O.pairwise_sum(y))) / y.size, 1.0 - float(y.max()))
    sref = O.newton_project_simplex(y, 1.0, lam0=lam0)
    d, a, b, l, u, r = p.instances.gen_cqk_arrays("cqk-correlated", 300007, 4)
    inst = p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
    ref = O.solve_cqk(d, a, b, l, u, r, fixing=True)
    Y = p.gen_simplex_y("simplex-n01", 64 * 512, 4).reshape(64, 512)
    X0 = np.asarray(p.project_simplex_rows(Y, 1.0)[0])

    def check_cqk(out):
        assert abs(out.lam - ref["lam"]) <= TOL * max(1.0, abs(ref["lam"]))
        assert out.fixed_count == ref["fixed_count"]

    def check_spx(out):
        assert abs(out.lam - sref["lam"]) <= TOL * max(1.0, abs(sref["lam"]))
        assert np.array_equal(out.x, np.maximum(0.0, y + out.lam))

    def check_rows(out):
        assert np.array_equal(np.asarray(out[0]), X0)

    steps = [(lambda: p.solve_cqk(inst), check_cqk),
             (lambda: p.newton_project_simplex(y, 1.0, start="tight"), check_spx),
             (lambda: p.project_simplex_rows(Y, 1.0), check_rows)]
    for k in range(12):
        call, check = steps[(k * 5) % 3]
        env = (None, "CQK_STATIC_FINAL", None, "CQK_MASTER_STEP")[k % 4]
        check(call() if env is None else _with_env(env, call))
