"""A/B of the CQK start at C2-like sizes: unfused (pass 0 + full first
scan), fused without the direction guess, fused with it.  Kernel time, best
of 8, per (family, seed, n).  Perf aid; one JSON line per instance."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_15910_b200 as P
from paper_2603_15910_b200 import _native as N

sizes = [int(float(s)) for s in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["5e6", "1e7", "2e7"])]
h = N.handle()
modes = [("unfused", 10**15, 0), ("fused", 4_000_000, 0), ("fused+guess", 4_000_000, 1)]
for n in sizes:
    for fam in ("cqk-uncorrelated", "cqk-weakly-correlated", "cqk-correlated"):
        for seed in (1, 2, 3):
            inst = P.instances.gen_cqk_device(fam, n, seed)
            row = {"n": n, "family": fam, "seed": seed}
            best = {}
            for _ in range(6):  # modes interleaved: clock / thermal drift hits all alike
                for name, mn, g in modes:
                    h.set_fused(mn, 2e-3, g)
                    ms = P.solve_cqk(inst).stats["device_ms"]
                    best[name] = min(best.get(name, ms), ms)
            row.update({k: round(v, 4) for k, v in best.items()})
            h.set_fused(4_000_000, 2e-3, 1)
            print(json.dumps(row), flush=True)
