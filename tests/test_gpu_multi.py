"""Multi-device paths on whatever the box has: the C5 row split across
handles (spx_project_batched_multi_f64; several handles on cuda:0 stand in
for several GPUs, the per-row results must not depend on the split), local
groups across distinct GPUs (skipped on a one-GPU box), the grid-wide
timeout report of a collective whose peer never arrives, and the read-only
streaming peak used as the roofline's second denominator."""
import threading
import time

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("split", [2, 3])
def test_rows_split_across_handles_is_bit_identical(split):
    import paper_2603_15910_b200 as P

    rows, cols = 1001, 4096
    Y = P.gen_simplex_y("simplex-n01", rows * cols, 3).reshape(rows, cols)
    X1, lam1, it1, st1 = P.project_simplex_rows(Y, 1.0)
    Xm, lamm, itm, stm = P.project_simplex_rows(Y, 1.0, devices=[0] * split)
    assert np.array_equal(X1, Xm) and np.array_equal(lam1, lamm) and np.array_equal(it1, itm)
    assert stm["bytes_model"] == st1["bytes_model"]
    assert stm["launches"] == split
    for i in (0, 500, 1000):  # and the rows are the reference's projections
        ref = O.newton_project_simplex(Y[i], 1.0)
        assert abs(lamm[i] - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))
        assert np.abs(Xm[i] - ref["x"]).max() <= 1e-12


def test_rows_split_across_visible_gpus():
    import torch

    import paper_2603_15910_b200 as P

    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 visible GPUs")
    Y = P.gen_simplex_y("simplex-u01", 4096 * 2048, 5).reshape(4096, 2048)
    X1, lam1, _, _ = P.project_simplex_rows(Y, 1.0)
    Xm, lamm, _, _ = P.project_simplex_rows(Y, 1.0, devices=list(range(ngpu)))
    assert np.array_equal(X1, Xm) and np.array_equal(lam1, lamm)


def test_local_group_across_visible_gpus():
    """Same-process ranks on distinct devices: connect_local enables peer
    access, the kernels store into each other's mailboxes over NVLink."""
    import torch

    import paper_2603_15910_b200 as P
    from paper_2603_15910_b200 import distributed as D

    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 visible GPUs")
    world = min(ngpu, 8)
    n = 2_000_003
    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 4)
    ref = O.solve_cqk(d, a, b, l, u, r)
    comms = D.local_group(list(range(world)))
    solvers = []
    for q in range(world):
        lo, hi = D.shard_bounds(n, world, q)
        sh = [torch.from_numpy(v[lo:hi].copy()).cuda(q) for v in (d, a, b, l, u)]
        solvers.append(D.ShardedCQK(sh, r, n_total=n, offset=lo, comm=comms[q]))
    outs = [None] * world

    def work(q):
        torch.cuda.set_device(q)
        s = torch.cuda.Stream(q)
        with torch.cuda.stream(s):
            outs[q] = solvers[q].solve()
        s.synchronize()

    th = [threading.Thread(target=work, args=(q,)) for q in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert len({o.lam for o in outs}) == 1
    assert abs(outs[0].lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))
    assert outs[0].iterations == ref["iterations"]


def test_collective_without_peer_reports_timeout():
    """Rank 1 never launches: rank 0's kernel must give up after the spin
    timeout (4 s) and the call must fail loudly instead of hanging or
    returning a partial x."""
    import torch

    import paper_2603_15910_b200 as P
    from paper_2603_15910_b200 import _native as N
    from paper_2603_15910_b200 import distributed as D

    n = 300_000
    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-uncorrelated", n, 2)
    comms = D.local_group([0, 0], grid_limit=32)
    lo, hi = D.shard_bounds(n, 2, 0)
    sh = [torch.from_numpy(v[lo:hi].copy()).cuda() for v in (d, a, b, l, u)]
    s0 = D.ShardedCQK(sh, r, n_total=n, offset=lo, comm=comms[0])
    t0 = time.time()
    with pytest.raises(N.NativeError, match="timed out"):
        s0.solve()
    assert time.time() - t0 < 60
    # the handle stays usable for ordinary solves
    out = P.solve_cqk(P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r))
    assert out.status is P.Status.SOLVED


def test_read_peak_is_a_streaming_rate():
    import torch

    from paper_2603_15910_b200 import _native as N

    arrs = [torch.ones(1 << 25, dtype=torch.float64, device="cuda") for _ in range(5)]
    gbs, ms = N.handle(0).read_peak(arrs, reps=3)
    assert 2000.0 < gbs < 9000.0, gbs  # B200 HBM3e: ~7 TB/s read-only
    assert ms > 0
