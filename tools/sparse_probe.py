"""Dense vs output="sparse" time of the l1 projection (C4 sizes)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_15910_b200 as P

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
y = torch.from_numpy(P.gen_simplex_y("simplex-n01", n, 1)).cuda()
res = {}
for name, f in (("dense", lambda: P.project_l1(y, 1.0)), ("sparse", lambda: P.project_l1(y, 1.0, output="sparse"))):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    res[name + "_call_ms"] = min(ts) * 1e3
idx, val = P.project_l1(y, 1.0, output="sparse")
res["nnz"] = int(idx.numel())
print(json.dumps({"n": n, **res}))
