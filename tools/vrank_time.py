"""Device time of a 2-rank sharded solve on one GPU (virtual ranks, 74 CTAs
each): the multi-GPU protocol's per-epoch cost, master vs masterless grid
step (CQK_MASTER_STEP=1).  Perf aid; one JSON line."""
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_15910_b200 as P
from paper_2603_15910_b200 import distributed as D

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**7
world = 2
d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-uncorrelated", n, 7)
comms = D.local_group([0] * world, grid_limit=148 // world)
solvers = []
for q in range(world):
    lo, hi = D.shard_bounds(n, world, q)
    sh = [torch.from_numpy(v[lo:hi].copy()).cuda() for v in (d, a, b, l, u)]
    solvers.append(D.ShardedCQK(sh, r, n_total=n, offset=lo, comm=comms[q]))


def run():
    out = [None] * world

    def work(q):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            out[q] = solvers[q].solve()
        s.synchronize()

    th = [threading.Thread(target=work, args=(q,)) for q in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out


for _ in range(3):
    run()
ms = []
for _ in range(10):
    outs = run()
    ms.append(max(o.stats["device_ms"] for o in outs))
ms.sort()
print(json.dumps({"n": n, "world": world, "master_step": os.environ.get("CQK_MASTER_STEP", "0"),
                  "median_ms": ms[len(ms) // 2], "min_ms": ms[0], "evals": outs[0].phi_evals,
                  "lam": outs[0].lam}))
