"""Find random instances where the device solve's iterate sequence departs
from the oracle's (perf-iteration / debugging aid)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
import paper_2603_15910_b200 as P  # noqa: E402
from paper_2603_15910_b200 import newton as NW  # noqa: E402
from test_gpu_parity import random_arrays  # noqa: E402

bad = 0
for seed in range(120):
    d, a, b, l, u, r = random_arrays(seed, 1 + seed % 60)
    inst = P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
    tr = []
    out = NW.run_cqk(inst, P.SolverOptions(variable_fixing=True), NW.N.VARIANT_SOLVE, trace=tr)
    ref = O.solve_cqk(d, a, b, l, u, r, fixing=True)
    if ref["status"] != 0:
        continue
    if out.iterations != ref["iterations"] or out.phi_evals != ref["phi_evals"]:
        bad += 1
        print("seed", seed, "n", d.size, "its", out.iterations, ref["iterations"], "evals",
              out.phi_evals, ref["phi_evals"], "fixed", out.fixed_count, ref["fixed_count"])
        print("  device trace:", [tuple(float(v) for v in t) for t in tr])
print("mismatches", bad)
