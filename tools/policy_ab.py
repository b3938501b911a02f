"""A/B of the fused-start policies (direction guess, compaction ratio) over
instance families, sizes and seeds: kernel time and bytes per solve.
Perf aid; one JSON line per (size, family, seed)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2603_15910_b200 as P
from paper_2603_15910_b200 import _native as N

sizes = [int(float(s)) for s in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["5e6", "1e7", "3e7", "1e8"])]
fams = ["cqk-uncorrelated", "cqk-weakly-correlated", "cqk-correlated"]
policies = [("g0", 0, None), ("auto", 1, None)]
h = N.handle()
for n in sizes:
    for fam in fams:
        for seed in (1, 2, 3):
            inst = P.instances.gen_cqk_device(fam, n, seed)
            row = {"n": n, "family": fam, "seed": seed}
            for name, g, cr in policies:
                h.set_fused(4_000_000, 2e-3, g)
                opts = P.SolverOptions(compact_ratio=cr)
                best = None
                for _ in range(4):
                    out = P.solve_cqk(inst, opts)
                    ms = out.stats["device_ms"]
                    best = ms if best is None else min(best, ms)
                row[name] = [round(best, 4), round(out.stats["bytes_model"] / n, 1), out.phi_evals]
            h.set_fused(4_000_000, 2e-3, 1)
            print(json.dumps(row), flush=True)
            del inst
            torch.cuda.empty_cache()
