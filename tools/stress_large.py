"""Parity at the configs' scale: random CQK instances n in [1e7, 1e8] (the
fused start, the direction guess and the compaction policy all active) solved
by solve_cqk on the device and by the oracle's restatement of
newton.py:209-342 on the host (test infrastructure as the checker).
Compares lambda (1e-12 relative), x (1e-12 scaled), feasibility (beside
the oracle's own: both stop at tau = eps^0.75, newton.py:64-67),
iterations, phi evaluations and fixed counts; writes
gpurun_out/stress_large.json.  Usage: python tools/stress_large.py [count]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle as O
import paper_2603_15910_b200 as P

count = int(sys.argv[1]) if len(sys.argv) > 1 else 24
rng = np.random.default_rng(2028)
rows, worst_lam, worst_x = [], 0.0, 0.0
t0 = time.time()
for k in range(count):
    n = int(10 ** rng.uniform(7.0, 8.0))
    fam = O.CQK_FAMILIES[k % 3]
    seed = 7000 + k
    d, a, b, l, u, r = O.gen_cqk(fam, n, seed)
    level = None
    if k % 4 == 3:  # a different right-hand side: b.l + U (b.u - b.l)
        level = float(rng.choice([0.02, 0.3, 0.7, 0.98]))
        bl, bu = float(O.pairwise_sum(b * l)), float(O.pairwise_sum(b * u))
        r = bl + level * (bu - bl)
    ref = O.solve_cqk(d, a, b, l, u, r)
    inst = P.CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r)
    out = P.solve_cqk(inst)
    x = out.x.cpu().numpy()
    rel = abs(out.lam - ref["lam"]) / max(1.0, abs(ref["lam"]))
    xs = float(np.abs(x - ref["x"]).max()) / max(1.0, float(np.abs(ref["x"]).max()))
    bx = b * x
    feas = abs(float(O.pairwise_sum(bx)) - r) / float(O.pairwise_sum(np.abs(bx)))
    bxr = b * ref["x"]  # the reference algorithm's own residual (it stops at tau = eps^0.75)
    feas_ref = abs(float(O.pairwise_sum(bxr)) - r) / float(O.pairwise_sum(np.abs(bxr)))
    worst_lam, worst_x = max(worst_lam, rel), max(worst_x, xs)
    row = {"family": fam, "n": n, "seed": seed, "r_level": level, "lam_rel": rel, "x_scaled": xs,
           "feas_rel": feas, "feas_rel_oracle": feas_ref, "iterations": [out.iterations, ref["iterations"]],
           "phi_evals": [out.phi_evals, ref["phi_evals"]],
           "fixed_count": [out.fixed_count, ref["fixed_count"]],
           "device_ms": out.stats["device_ms"]}
    rows.append(row)
    print(json.dumps(row), flush=True)
    del inst, out, x, d, a, b, l, u, ref
    torch.cuda.empty_cache()
ok = all(r_["lam_rel"] <= 1e-12 and r_["x_scaled"] <= 1e-12 for r_ in rows)
same = sum(r_["iterations"][0] == r_["iterations"][1] and r_["phi_evals"][0] == r_["phi_evals"][1]
           and r_["fixed_count"][0] == r_["fixed_count"][1] for r_ in rows)
summary = {"instances": len(rows), "n_range": [min(r_["n"] for r_ in rows), max(r_["n"] for r_ in rows)],
           "lam_worst_rel": worst_lam, "x_worst_scaled": worst_x,
           "feas_worst_rel": max(r_["feas_rel"] for r_ in rows),
           "feas_worst_rel_oracle": max(r_["feas_rel_oracle"] for r_ in rows),
           "identical_iterations_evals_fixed": same, "all_within_1e-12": ok, "wall_s": time.time() - t0,
           "rows": rows}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "stress_large.json"), "w") as f:
    json.dump(summary, f, indent=1)
print(json.dumps({k: v for k, v in summary.items() if k != "rows"}))
sys.exit(0 if ok else 1)
