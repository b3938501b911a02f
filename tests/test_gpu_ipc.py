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


def _worker(rank, world, port, q, per_gpu=False):
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
        dev = rank if per_gpu else 0  # one process per visible GPU, or all on cuda:0
        torch.cuda.set_device(dev)
        h = N.Handle(dev)
        if not per_gpu:
            h.lib.cqk_set_grid_limit(h.ptr, 16)
        comm = D.Communicator(h, rank, world)  # IPC handles over gloo
        sh = [torch.from_numpy(v[lo:hi].copy()).cuda(dev) for v in (d, a, b, l, u)]
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


def _run(world, per_gpu):
    import oracle as O
    import paper_2603_15910_b200 as P

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, per_gpu)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    assert all(len(t) == 6 for t in res), res
    n = 200_003
    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 11)
    ref = O.solve_cqk(d, a, b, l, u, r)
    assert len({t[1] for t in res}) == 1  # the identical decision on every rank
    assert abs(res[0][1] - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))
    assert res[0][2] == ref["iterations"] and res[0][3] == ref["fixed_count"]
    x = np.concatenate([t[5] for t in res])
    assert np.abs(x - ref["x"]).max() <= 1e-12 * 25


def test_ipc_two_processes():
    _run(2, per_gpu=False)


def test_ipc_one_process_per_gpu():
    """The deployment shape: one process per visible GPU, mailboxes mapped
    over CUDA IPC with peer access (NVLink) -- skipped on a one-GPU box."""
    import torch

    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 visible GPUs")
    _run(min(ngpu, 8), per_gpu=True)
