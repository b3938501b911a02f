"""Host-side logic of the multi-GPU path on CPU: world-size-2 gloo process
group exercising the shard partition, the one-time handle exchange and the
sharded instance generation + rank-order r (no device compute)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_15910_b200 as P
        from paper_2603_15910_b200.distributed import allgather_bytes, shard_bounds

        blobs = allgather_bytes(bytes([rank]) * 64)
        assert [b[0] for b in blobs] == list(range(world))
        n = 100_003
        lo, hi = shard_bounds(n, world, rank)
        d, a, b, l, u, bl, bu = P.instances.gen_cqk_shard("cqk-weakly-correlated", n, 9, lo, hi)
        parts = [np.frombuffer(x) for x in allgather_bytes(np.array([bl, bu]).tobytes())]
        sbl = sum(p[0] for p in parts)
        sbu = sum(p[1] for p in parts)
        r = P.instances.cqk_r("cqk-weakly-correlated", n, 9, sbl, sbu)
        full = P.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 9)
        same = all(np.array_equal(x, y[lo:hi]) for x, y in zip((d, a, b, l, u), full[:5]))
        rs = allgather_bytes(np.array([r]).tobytes())
        q.put((rank, same, len(set(rs)) == 1, abs(r - full[5]) / abs(full[5])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, r_agree, r_rel in res:
        assert same, rank
        assert r_agree
        assert r_rel < 1e-14


def test_shard_bounds_cover():
    from paper_2603_15910_b200.distributed import shard_bounds

    for n in (1, 7, 100, 10**8 + 3):
        for w in (1, 2, 3, 8):
            b = [shard_bounds(n, w, q) for q in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[q][1] == b[q + 1][0] for q in range(w - 1))
