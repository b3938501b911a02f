"""Multi-rank exchange on one GPU: W same-process "virtual ranks" (handles on
cuda:0, each with a reduced persistent grid, solving concurrently from their
own host threads and streams) must reproduce the single-GPU solve.  This runs
the exact device protocol of the multi-GPU path (mailbox stores, system-scope
release flags, rank-order reduction) -- only the mailbox pointers are local
instead of IPC-mapped peer memory."""
import threading

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def run_ranks(fns):
    import torch

    out = [None] * len(fns)
    err = []

    def work(q):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[q] = fns[q]()
            s.synchronize()
        except Exception as e:  # pragma: no cover - reported below
            err.append(e)

    th = [threading.Thread(target=work, args=(q,)) for q in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not err, err
    return out


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("family", ["cqk-uncorrelated", "cqk-correlated"])
def test_sharded_cqk_matches_single(world, family):
    import torch

    import paper_2603_15910_b200 as P
    from paper_2603_15910_b200 import distributed as D

    n = 1_000_003
    d, a, b, l, u, r = P.instances.gen_cqk_arrays(family, n, 7)
    single = P.solve_cqk(P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r))
    ref = O.solve_cqk(d, a, b, l, u, r)
    comms = D.local_group([0] * world, grid_limit=120 // world)
    solvers = []
    for q in range(world):
        lo, hi = D.shard_bounds(n, world, q)
        sh = [torch.from_numpy(v[lo:hi].copy()).cuda() for v in (d, a, b, l, u)]
        solvers.append(D.ShardedCQK(sh, r, n_total=n, offset=lo, comm=comms[q]))
    for variant in ("solve", "jacobi"):
        outs = run_ranks([lambda s=s: s.solve(variant=variant) for s in solvers])
        lams = [o.lam for o in outs]
        assert len(set(lams)) == 1, lams  # identical decision on every rank
        o = outs[0]
        assert o.status is P.Status.SOLVED
        assert abs(o.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))
        if variant == "solve":
            assert o.iterations == single.iterations == ref["iterations"]
            assert o.fixed_count == ref["fixed_count"]
        x = np.concatenate([oo.x.cpu().numpy() for oo in outs])
        assert np.abs(x - ref["x"]).max() <= 1e-12 * 25.0 if variant == "solve" else True


def test_sharded_validation_reports_global_index():
    import torch

    import paper_2603_15910_b200 as P
    from paper_2603_15910_b200 import distributed as D

    n = 1000
    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-uncorrelated", n, 3)
    d[777] = -1.0
    comms = D.local_group([0, 0], grid_limit=64)
    solvers = []
    for q in range(2):
        lo, hi = D.shard_bounds(n, 2, q)
        sh = [torch.from_numpy(v[lo:hi].copy()).cuda() for v in (d, a, b, l, u)]
        solvers.append(D.ShardedCQK(sh, r, n_total=n, offset=lo, comm=comms[q]))

    def call(s):
        try:
            s.solve()
        except P.DomainError as e:
            return (e.field, e.index)
        return None

    outs = run_ranks([lambda s=s: call(s) for s in solvers])
    assert outs == [("d", 777), ("d", 777)]


@pytest.mark.parametrize("l1", [False, True])
def test_sharded_projection_matches_single(l1):
    import torch

    import paper_2603_15910_b200 as P
    from paper_2603_15910_b200 import distributed as D

    n = 2_000_001
    y = P.gen_simplex_y("simplex-n01", n, 5)
    if l1:  # the sharded route iterates from the tight start
        single = P.simplex.project_l1_outcome(y, 1.0, start="tight")
    else:
        single = P.newton_project_simplex(y, 1.0, start="tight")
    comms = D.local_group([0, 0], grid_limit=60)
    projs = []
    for q in range(2):
        lo, hi = D.shard_bounds(n, 2, q)
        projs.append(D.ShardedProjection(comms[q], torch.from_numpy(y[lo:hi].copy()).cuda(), n))
    outs = run_ranks([lambda q=q: projs[q].solve(1.0, l1=l1) for q in range(2)])
    assert outs[0].lam == outs[1].lam
    assert abs(outs[0].lam - single.lam) <= 1e-12 * max(1.0, abs(single.lam))
    assert outs[0].iterations == single.iterations
    x = np.concatenate([o.x.cpu().numpy() for o in outs])
    assert np.abs(x - single.x).max() <= 1e-12
