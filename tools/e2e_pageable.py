"""Public-API host solves from ordinary (pageable) numpy arrays -- the way a
reference caller passes data -- vs pinned arrays (perf-iteration aid)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15910_b200 as P  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 1)
for kind in ("pageable", "pinned"):
    arrs = [d, a, b, l, u] if kind == "pageable" else [torch.from_numpy(v).pin_memory().numpy() for v in (d, a, b, l, u)]
    inst = P.CqkInstance(*arrs, r=r)
    for _ in range(2):
        out = P.solve_cqk(inst)
        del out
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        out = P.solve_cqk(inst)
        ts.append(time.perf_counter() - t0)
        del out
    print(json.dumps({"inputs": kind, "n": n, "ms": 1e3 * min(ts), "elements_per_s": n / min(ts)}), flush=True)
