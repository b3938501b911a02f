"""C5 timing (65536 x 4096 N(0,1), r = 1): device time per launch (the
library's own CUDA events), fraction of the copy peak, rerun identity."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15910_b200 as P  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
g = torch.Generator(device="cuda").manual_seed(1)
Y = torch.randn(rows, cols, dtype=torch.float64, device="cuda", generator=g)
ts, first = [], None
for i in range(20):
    X, lam, its, st = P.project_simplex_rows(Y, 1.0)
    ts.append(st["device_ms"])
    if first is None:
        first = (X.clone(), lam.clone())
torch.cuda.synchronize()
best, med = min(ts[3:]), sorted(ts[3:])[len(ts[3:]) // 2]
gbs = 16 * rows * cols / (best * 1e-3) / 1e9
print(json.dumps({"rows": rows, "cols": cols, "best_ms": best, "median_ms": med, "GBps_best": gbs,
                  "frac_copy": gbs / 6547.2, "iters_mean": float(its.double().mean()),
                  "rerun_identical": bool(torch.equal(X, first[0]) and torch.equal(lam, first[1])),
                  "row_sum_err": float((X.sum(1) - 1).abs().max())}))
