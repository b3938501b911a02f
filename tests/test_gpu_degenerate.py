"""Rare paths of the solve state machine (newton.py:129-162, 280-326) on the
engine that serves production sizes -- the TMA pipeline, n >= 64Ki per rank
-- and through the sharded MIN/MAX exchange of 2-3 virtual ranks, against
the C oracle: plateaus where phi' = 0 forces the nearest-breakpoint search
(both directions, with and without fixing), a replicated pinned box that is
INFEASIBLE (test_newton.py:114-118, test_parallel.py:80-83 scaled up),
l == u blocks mixed into random instances, and MaxIterationsError."""
import threading

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

from degenerate_cases import CASES, N  # noqa: E402


def P():
    import paper_2603_15910_b200 as p

    return p


@pytest.fixture(autouse=True)
def tma_engine():
    from paper_2603_15910_b200 import _native as Nn

    h = Nn.handle()
    h.lib.cqk_set_engine(h.ptr, 1)
    yield
    h.lib.cqk_set_engine(h.ptr, 0)


def check(out, ref, x=None):
    p = P()
    if ref["status"] == O.INFEASIBLE:
        assert out.status is p.Status.INFEASIBLE and out.lam is None and out.x is None
    else:
        assert out.status is p.Status.SOLVED and ref["status"] == O.SOLVED
        assert abs(out.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"])), (out.lam, ref["lam"])
        xx = out.x.cpu().numpy() if x is None else x
        assert np.abs(xx - ref["x"]).max() <= 1e-12 * max(1.0, np.abs(ref["x"]).max())
    assert out.iterations == ref["iterations"], (out.iterations, ref["iterations"])
    assert out.phi_evals == ref["phi_evals"]
    assert out.fixed_count == ref["fixed_count"]


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("fixing", [True, False])
def test_degenerate_single_gpu(case, fixing):
    import torch

    p = P()
    d, a, b, l, u, r = CASES[case]()
    ref = O.solve_cqk(d, a, b, l, u, r, fixing=fixing)
    inst = p.CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r)
    out = p.solve_cqk(inst, p.SolverOptions(variable_fixing=fixing))
    check(out, ref)
    if case.startswith("plateau"):
        assert ref["iterations"] >= 2  # the breakpoint jump was taken


@pytest.mark.parametrize("case", sorted(CASES))
def test_degenerate_jacobi(case):
    import torch

    p = P()
    d, a, b, l, u, r = CASES[case]()
    ref = O.jacobi_solve(d, a, b, l, u, r)
    inst = p.CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r)
    check(p.jacobi_solve(inst), ref)


def test_max_iterations_on_tma_engine():
    p = P()
    d, a, b, l, u, r = O.gen_cqk("cqk-weakly-correlated", N, 4)
    ref = O.solve_cqk(d, a, b, l, u, r, max_iter=1)
    assert ref["status"] == O.E_MAXITER
    import torch

    inst = p.CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r)
    with pytest.raises(p.MaxIterationsError) as ei:
        p.solve_cqk(inst, p.SolverOptions(max_iterations=1))
    assert ei.value.iterations == ref["iterations"] and ei.value.phi_evals == ref["phi_evals"]
    assert abs(ei.value.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))


def _sharded(case_arrays, world, variant):
    import torch

    from paper_2603_15910_b200 import distributed as D

    d, a, b, l, u, r = case_arrays
    n = d.size
    comms = D.local_group([0] * world, grid_limit=120 // world)
    for c in comms:
        c.handle.lib.cqk_set_engine(c.handle.ptr, 1)
    solvers = []
    for q in range(world):
        lo, hi = D.shard_bounds(n, world, q)
        sh = [torch.from_numpy(v[lo:hi].copy()).cuda() for v in (d, a, b, l, u)]
        solvers.append(D.ShardedCQK(sh, r, n_total=n, offset=lo, comm=comms[q]))
    outs, err = [None] * world, []

    def work(q):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                outs[q] = solvers[q].solve(variant=variant)
                if outs[q].x is not None:
                    outs[q] = (outs[q], outs[q].x.cpu().numpy())
                else:
                    outs[q] = (outs[q], None)
            s.synchronize()
        except Exception as e:  # pragma: no cover
            err.append(e)

    th = [threading.Thread(target=work, args=(q,)) for q in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not err, err
    return outs


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("world", [2, 3])
def test_degenerate_sharded(case, world):
    """The breakpoint MIN / MAX and the infeasible verdict through the
    in-kernel exchange: every rank takes the oracle's decisions."""
    arrays = CASES[case]()
    d, a, b, l, u, r = arrays
    for variant, ref in (("solve", O.solve_cqk(d, a, b, l, u, r)), ("jacobi", O.jacobi_solve(d, a, b, l, u, r))):
        outs = _sharded(arrays, world, variant)
        assert len({(o.status, o.lam, o.iterations) for o, _ in outs}) == 1
        x = None if outs[0][1] is None else np.concatenate([xx for _, xx in outs])
        check(outs[0][0], ref, x=x)
