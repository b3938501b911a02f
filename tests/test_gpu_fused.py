"""The fused start of the TMA CQK solve (cqk_tma.cuh: sample pass, fused
lambda0 + validate + classification pass, side-list first scan) against the
oracle and against the unfused solve (pass 0 + a full first scan):

* random instances of the three families, solve and Jacobi, with the default
  interval, a zero-width interval (lambda0 always outside: the full first
  scan after the fused pass) and a very wide one (most elements in the side
  list);
* the degenerate instances (plateaus and breakpoint searches, the pinned
  INFEASIBLE box, l == u blocks, MaxIterations) through the fused start;
* every validate() check (core.py:126-165): the first failing check in the
  reference's order and its first offending index;
* 2 and 3 virtual ranks (the fused totals cross the in-kernel exchange);
* the direction guess (cqk_set_fused_guess): auto, off, and both forced
  directions -- one of which is wrong and must simply not be adopted."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

from degenerate_cases import CASES  # noqa: E402

OFF = 10**18


def P():
    import paper_2603_15910_b200 as p

    return p


def handle():
    from paper_2603_15910_b200 import _native as Nn

    return Nn.handle()


@pytest.fixture(autouse=True)
def restore():
    h = handle()
    h.lib.cqk_set_engine(h.ptr, 1)
    yield
    h.lib.cqk_set_engine(h.ptr, 0)
    h.set_fused(4_000_000, 2e-3)


def solve(inst, fused, width=2e-3, guess=1, **kw):
    p = P()
    handle().set_fused(0 if fused else OFF, width, guess)
    if kw.pop("jacobi", False):
        return p.jacobi_solve(inst, p.SolverOptions(**kw))
    return p.solve_cqk(inst, p.SolverOptions(**kw))


def check(out, ref):
    p = P()
    if ref["status"] == O.INFEASIBLE:
        assert out.status is p.Status.INFEASIBLE
    else:
        assert out.status is p.Status.SOLVED and ref["status"] == O.SOLVED
        assert abs(out.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"])), (out.lam, ref["lam"])
        x = out.x.cpu().numpy()
        assert np.abs(x - ref["x"]).max() <= 1e-12 * max(1.0, np.abs(ref["x"]).max())
    assert out.iterations == ref["iterations"], (out.iterations, ref["iterations"])
    assert out.phi_evals == ref["phi_evals"]
    assert out.fixed_count == ref["fixed_count"]


def inst_of(d, a, b, l, u, r):
    import torch

    return P().CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r)


@pytest.mark.parametrize("family", ["cqk-uncorrelated", "cqk-weakly-correlated", "cqk-correlated"])
@pytest.mark.parametrize("width", [2e-3, 0.0, 0.5])
def test_fused_matches_oracle_and_unfused(family, width):
    p = P()
    for seed in (1, 2):
        n = 300_000 + 7 * seed
        d, a, b, l, u, r = p.instances.gen_cqk_arrays(family, n, seed)
        inst = inst_of(d, a, b, l, u, r)
        for jac in (False, True):
            ref = O.solve_cqk(d, a, b, l, u, r, fixing=not jac)
            f = solve(inst, True, width, jacobi=jac)
            g = solve(inst, False, jacobi=jac)
            check(f, ref)
            assert (f.iterations, f.phi_evals, f.fixed_count) == (g.iterations, g.phi_evals, g.fixed_count)
            assert abs(f.lam - g.lam) <= 1e-13 * max(1.0, abs(g.lam))


def test_fused_saves_pass0_bytes():
    """At a size where the sample (4 tiles per CTA) is a small fraction, the
    fused start moves ~24 B / element fewer than pass 0 + a full first scan."""
    p = P()
    n = 5_000_000
    d, a, b, l, u, r = p.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 3)
    inst = inst_of(d, a, b, l, u, r)
    f, g = solve(inst, True, guess=0), solve(inst, False)
    assert (f.iterations, f.phi_evals, f.fixed_count) == (g.iterations, g.phi_evals, g.fixed_count)
    saved = (g.stats["bytes_model"] - f.stats["bytes_model"]) / n
    assert 15.0 < saved <= 24.0, saved


@pytest.mark.parametrize("family", ["cqk-uncorrelated", "cqk-weakly-correlated", "cqk-correlated"])
@pytest.mark.parametrize("guess", [0, 1, 2, 3])
def test_fused_direction_guess(family, guess):
    """Every guess mode returns the oracle's solve; the iterate sequence is
    that of the unfused solve (only the summation order may differ)."""
    p = P()
    for seed in (1, 2, 3):
        n = 400_000 + 11 * seed
        d, a, b, l, u, r = p.instances.gen_cqk_arrays(family, n, seed)
        inst = inst_of(d, a, b, l, u, r)
        ref = O.solve_cqk(d, a, b, l, u, r)
        f = solve(inst, True, guess=guess)
        g = solve(inst, False)
        check(f, ref)
        assert (f.iterations, f.phi_evals, f.fixed_count) == (g.iterations, g.phi_evals, g.fixed_count)


def test_fused_guess_saves_the_first_reread():
    """weak, n = 1e7, seed 1 (sampled residual ~8% of sum|bx|: the guess
    fires): the confirmed guess replaces the second full read (40 B) by the
    survivors' write and read."""
    p = P()
    n = 10_000_000
    d, a, b, l, u, r = p.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 1)
    inst = inst_of(d, a, b, l, u, r)
    f, g = solve(inst, True, guess=1), solve(inst, True, guess=0)
    assert (f.iterations, f.phi_evals, f.fixed_count) == (g.iterations, g.phi_evals, g.fixed_count)
    assert f.stats["bytes_model"] < g.stats["bytes_model"], (f.stats, g.stats)


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("fixing", [True, False])
@pytest.mark.parametrize("guess", [1, 2, 3])
def test_fused_degenerate(case, fixing, guess):
    d, a, b, l, u, r = CASES[case]()
    ref = O.solve_cqk(d, a, b, l, u, r, fixing=fixing)
    p = P()
    try:
        out = solve(inst_of(d, a, b, l, u, r), True, guess=guess, variable_fixing=fixing)
    except p.MaxIterationsError:
        assert ref["status"] == O.E_MAXITER
        return
    check(out, ref)


# (array, value, field) in validate()'s order: d/a/b finite, l/u NaN, d > 0,
# b > 0, l <= u, l != +inf, u != -inf
BAD = [("d", np.inf, "d"), ("a", np.nan, "a"), ("b", -np.inf, "b"), ("l", np.nan, "l"),
       ("u", np.nan, "u"), ("d", -2.0, "d"), ("b", 0.0, "b"), ("l", 1e9, "l"),
       ("l", np.inf, "l"), ("u", -np.inf, "u")]


@pytest.mark.parametrize("k", range(len(BAD)))
def test_fused_validation_first_check_first_index(k):
    p = P()
    n = 250_000
    arrs = dict(zip("dabluv", p.instances.gen_cqk_arrays("cqk-uncorrelated", n, 5)))
    r = arrs.pop("v")
    rng = np.random.default_rng(k)
    name, val, field = BAD[k]
    pos = np.sort(rng.choice(n, 3, replace=False))
    for i in pos:
        arrs[name][i] = val
    if k == 7:  # l > u needs l below +inf
        arrs["u"][pos] = 0.0
    later = int(rng.integers(0, n))  # a later check class failing earlier must not win
    arrs["d"][later] = -1.0 if k < 5 else arrs["d"][later]
    inst = inst_of(arrs["d"], arrs["a"], arrs["b"], arrs["l"], arrs["u"], r)
    seen = []
    for fused in (True, False):
        try:
            solve(inst, fused)
            seen.append(None)
        except p.DomainError as e:
            seen.append((e.field, e.index))
    assert seen[0] == seen[1], seen
    if k < 5:
        assert seen[0] == (field, int(pos[0]))


def run_ranks(fns):
    """Each virtual rank on its own host thread and stream (test_gpu_sharded.py)."""
    from test_gpu_sharded import run_ranks as rr

    return rr(fns)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("guess", [1, 2, 3])
def test_fused_sharded(world, guess):
    import torch

    p = P()
    from paper_2603_15910_b200 import distributed as D

    n = 600_011
    d, a, b, l, u, r = p.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 9)
    ref = O.solve_cqk(d, a, b, l, u, r)
    comms = D.local_group([0] * world, grid_limit=120 // world)
    solvers = []
    for q in range(world):
        comms[q].handle.set_fused(0, 2e-3, guess)
        lo, hi = D.shard_bounds(n, world, q)
        sh = [torch.from_numpy(v[lo:hi].copy()).cuda() for v in (d, a, b, l, u)]
        solvers.append(D.ShardedCQK(sh, r, n_total=n, offset=lo, comm=comms[q]))
    outs = run_ranks([lambda s=s: s.solve() for s in solvers])
    assert len({o.lam for o in outs}) == 1
    o = outs[0]
    assert abs(o.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))
    assert (o.iterations, o.phi_evals, o.fixed_count) == (ref["iterations"], ref["phi_evals"],
                                                          ref["fixed_count"])
    x = np.concatenate([oo.x.cpu().numpy() for oo in outs])
    assert np.abs(x - ref["x"]).max() <= 1e-12 * 25.0


@pytest.mark.parametrize("guess", [0, 1, 2, 3])
def test_fused_infinite_bounds(guess):
    """l = -inf / u = +inf entries (allowed by validate, core.py:126-165): never
    classified at a bound, never fixed there; the fused start with every
    guess mode returns the oracle's solve."""
    p = P()
    n = 400_003
    d, a, b, l, u, r = p.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 21)
    rng = np.random.default_rng(21)
    l = l.copy()
    u = u.copy()
    l[rng.random(n) < 0.2] = -np.inf
    u[rng.random(n) < 0.2] = np.inf
    ref = O.solve_cqk(d, a, b, l, u, r)
    out = solve(inst_of(d, a, b, l, u, r), True, guess=guess)
    check(out, ref)
