"""Diagnose same-GPU virtual ranks: kernel start times per rank."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2603_15910_b200 as P
from paper_2603_15910_b200 import distributed as D

grid = int(sys.argv[1])
n = int(float(sys.argv[2]))
prior = sys.argv[3] == "1"
d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-uncorrelated", n, 7)
if prior:
    print("single", P.solve_cqk(P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)).lam)
comms = D.local_group([0, 0], grid_limit=grid)
fused_min = int(float(os.environ.get("DIAG_FUSED_MIN", "1e18")))
for c in comms:
    c.handle.set_fused(fused_min, 2e-3)
solvers = []
for q in range(2):
    lo, hi = D.shard_bounds(n, 2, q)
    sh = [torch.from_numpy(v[lo:hi].copy()).cuda() for v in (d, a, b, l, u)]
    solvers.append(D.ShardedCQK(sh, r, n_total=n, offset=lo, comm=comms[q]))
res = [None, None]


def work(q):
    s = torch.cuda.Stream()
    t0 = time.time()
    try:
        with torch.cuda.stream(s):
            res[q] = ("ok", solvers[q].solve().lam, time.time() - t0)
    except Exception as e:
        res[q] = ("err", str(e), time.time() - t0)


th = [threading.Thread(target=work, args=(q,)) for q in range(2)]
[t.start() for t in th]
[t.join() for t in th]
print("grid", grid, "n", n, "prior", prior, res)
for q in range(2):
    tl = solvers[q].handle.timeline(12)
    print("rank", q, "start", tl[0, 3], [tuple(int(v) for v in row[:4]) for row in tl[1:10]])
