"""Kernel time vs n for both engines (CQK_ENGINE=tma|seg): the small-n
crossover of the TMA streaming engine (perf-iteration aid)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15910_b200 as P  # noqa: E402


def best(f, reps=10):
    for _ in range(3):
        f()
    return min(f().stats["device_ms"] for _ in range(reps))


for n in (10**5, 10**6, 3 * 10**6, 10**7, 3 * 10**7):
    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-uncorrelated", n, 1)
    inst = P.CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r)
    y = torch.from_numpy(P.gen_simplex_y("simplex-u01", n, 1)).cuda()
    print(json.dumps({"n": n, "cqk_ms": best(lambda: P.solve_cqk(inst)),
                      "spx_ms": best(lambda: P.newton_project_simplex(y, 1.0))}), flush=True)
