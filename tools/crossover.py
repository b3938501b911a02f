"""Engine crossover: device time of the TMA and the segment CQK engines over
n (perf aid for the CQK_TMA_MIN_N default).  One JSON line per (family, n)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2603_15910_b200 as P
from paper_2603_15910_b200 import _native as N

fams = {"unc": "cqk-uncorrelated", "weak": "cqk-weakly-correlated", "corr": "cqk-correlated"}
sizes = [int(float(s)) for s in (sys.argv[1:] or ["5e5", "1e6", "2e6", "4e6", "8e6", "1.6e7"])]
h = N.handle()
for fk, fam in fams.items():
    for n in sizes:
        d, a, b, l, u, r = P.instances.gen_cqk_arrays(fam, n, 1)
        inst = P.CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r)
        row = {"fam": fk, "n": n}
        for eng, code in (("tma", 1), ("seg", 2)):
            h.lib.cqk_set_engine(h.ptr, code)
            for _ in range(3):
                out = P.solve_cqk(inst)
            ts = []
            for _ in range(10):
                out = P.solve_cqk(inst)
                ts.append(out.stats["device_ms"])
            ts.sort()
            row[eng] = round(ts[len(ts) // 2] * 1e3, 1)
            row[eng + "_evals"] = out.phi_evals
        h.lib.cqk_set_engine(h.ptr, 0)
        print(json.dumps(row), flush=True)
