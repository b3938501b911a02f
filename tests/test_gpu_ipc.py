"""The multi-process path: two processes on one GPU exchange CUDA IPC mailbox
handles over a gloo process group and solve collectively (the kernels of the
two contexts time-slice, so this checks correctness, not speed)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_15910_b200 as P
        from paper_2603_15910_b200 import _native as N
        from paper_2603_15910_b200 import distributed as D

        n = 200_003
        d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 11)
        lo, hi = D.shard_bounds(n, world, rank)
        h = N.Handle(0)
        h.lib.cqk_set_grid_limit(h.ptr, 16)
        comm = D.Communicator(h, rank, world)  # IPC handles over gloo
        sh = [torch.from_numpy(v[lo:hi].copy()).cuda() for v in (d, a, b, l, u)]
        solver = D.ShardedCQK(sh, r, n_total=n, offset=lo, comm=comm)
        out = solver.solve()
        # the same collective solve from host memory (H2D / D2H in the library)
        oh = solver.solve_host([v[lo:hi] for v in (d, a, b, l, u)])
        assert oh.lam == out.lam and oh.iterations == out.iterations
        assert np.array_equal(oh.x, out.x.cpu().numpy())
        q.put((rank, out.lam, out.iterations, out.fixed_count, lo, out.x.cpu().numpy()))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_ipc_two_processes():
    import oracle as O
    import paper_2603_15910_b200 as P

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    assert all(len(t) == 6 for t in res), res
    n = 200_003
    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 11)
    ref = O.solve_cqk(d, a, b, l, u, r)
    assert res[0][1] == res[1][1]
    assert abs(res[0][1] - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))
    assert res[0][2] == ref["iterations"] and res[0][3] == ref["fixed_count"]
    x = np.concatenate([res[0][5], res[1][5]])
    assert np.abs(x - ref["x"]).max() <= 1e-12 * 25
