"""Quick device-time sweep over the hot-path workloads (perf iteration aid;
bench.py is the contract).  Prints one JSON line per workload."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2603_15910_b200 as P

PEAK = 6544.3
which = sys.argv[1:] or ["weak", "corr", "unc7", "jac", "spx", "l1", "rows"]


def timeit(f, reps=10):
    for _ in range(3):
        out = f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def cqk(fam, n, jac=False, ratio=None):
    d, a, b, l, u, r = P.instances.gen_cqk_arrays(fam, n, 1)
    inst = P.CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r)
    opts = P.SolverOptions(compact_ratio=ratio)
    f = (lambda: P.jacobi_solve(inst)) if jac else (lambda: P.solve_cqk(inst, opts))
    ms, out = timeit(f)
    st = out.stats
    return {"ms": ms, "kernel_ms": st["device_ms"], "GBps": st["bytes_model"] / st["device_ms"] / 1e6,
            "frac": st["bytes_model"] / st["device_ms"] / 1e6 / PEAK, "evals": out.phi_evals,
            "elem_per_s": n / ms * 1e3, "bytes_per_elem": st["bytes_model"] / n,
            "lam": out.lam, "iterations": out.iterations, "fixed": out.fixed_count}


res = {}
for w in which:
    if w == "weak":
        res[w] = cqk("cqk-weakly-correlated", 10**8)
    elif w == "weak_nocompact":
        res[w] = cqk("cqk-weakly-correlated", 10**8, ratio=2.0)
    elif w == "weak_always":
        res[w] = cqk("cqk-weakly-correlated", 10**8, ratio=0.0)
    elif w == "corr":
        res[w] = cqk("cqk-correlated", 10**8)
    elif w == "unc7":
        res[w] = cqk("cqk-uncorrelated", 10**7)
    elif w == "weak7":
        res[w] = cqk("cqk-weakly-correlated", 10**7)
    elif w == "unc6":
        res[w] = cqk("cqk-uncorrelated", 10**6)
    elif w == "weak6":
        res[w] = cqk("cqk-weakly-correlated", 10**6)
    elif w == "unc8":
        res[w] = cqk("cqk-uncorrelated", 10**8)
    elif w == "jac":
        res[w] = cqk("cqk-weakly-correlated", 10**8, jac=True)
    elif w == "weak_f32":  # the float32 path (warp-segment kernel, float element math)
        d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-weakly-correlated", 10**8, 1)
        inst = P.CqkInstance(*[torch.from_numpy(v.astype(np.float32)).cuda() for v in (d, a, b, l, u)], r=r)
        ms, out = timeit(lambda: P.solve_cqk(inst))
        st = out.stats
        res[w] = {"ms": ms, "kernel_ms": st["device_ms"], "GBps": st["bytes_model"] / st["device_ms"] / 1e6,
                  "frac": st["bytes_model"] / st["device_ms"] / 1e6 / PEAK, "evals": out.phi_evals,
                  "elem_per_s": 10**8 / ms * 1e3, "bytes_per_elem": st["bytes_model"] / 10**8}
    elif w.split("_")[0] in ("spx", "l1") and not w.startswith("spx1e6"):
        n = 10**8
        start = w.split("_")[1] if "_" in w else "auto"
        y = torch.from_numpy(P.gen_simplex_y("simplex-n01", n, 1)).cuda()
        if w.startswith("spx"):
            ms, out = timeit(lambda: P.newton_project_simplex(y, 1.0, start=start))
            st = out.stats
            ev = out.phi_evals
        else:
            ms, out = timeit(lambda: P.simplex.project_l1_outcome(y, 1.0, start=start))
            st = out.stats
            ev = out.phi_evals
        res[w] = {"ms": ms, "kernel_ms": st["device_ms"], "GBps": st["bytes_model"] / st["device_ms"] / 1e6,
                  "frac": st["bytes_model"] / st["device_ms"] / 1e6 / PEAK, "evals": ev,
                  "elem_per_s": n / ms * 1e3, "bytes_per_elem": st["bytes_model"] / n}
    elif w.startswith("spx1e6"):
        parts = w.split("_")[1:]
        start = next((x for x in parts if x in ("tight", "formula", "alg2", "auto")), "auto")
        fam = "simplex-n01" if "n01" in parts else "simplex-u01"
        y = torch.from_numpy(P.gen_simplex_y(fam, 10**6, 1)).cuda()
        ms, out = timeit(lambda: P.newton_project_simplex(y, 1.0, start=start), reps=50)
        res[w] = {"ms": ms, "kernel_ms": out.stats["device_ms"], "evals": out.phi_evals,
                  "launches": out.stats["launches"]}
    elif w == "rows":
        rows, cols = 65536, 4096
        Y = torch.from_numpy(P.gen_simplex_y("simplex-n01", rows * cols, 1)).cuda().view(rows, cols)
        ms, out = timeit(lambda: P.project_simplex_rows(Y, 1.0))
        st = out[3]
        res[w] = {"ms": ms, "kernel_ms": st["device_ms"], "GBps": st["bytes_model"] / st["device_ms"] / 1e6,
                  "frac": st["bytes_model"] / st["device_ms"] / 1e6 / PEAK,
                  "mean_iters": float(out[2].float().mean()), "elem_per_s": rows * cols / ms * 1e3}
    print(json.dumps({w: res[w]}), flush=True)
