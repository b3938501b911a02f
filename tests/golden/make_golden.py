"""Generate golden fixtures from the REAL reference package (run in the build
container, where /root/reference exists; the GPU box never reads it).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]

Writes tests/golden/small.npz (hand-derived + randomized small instances with
full outputs) and tests/golden/generated.json (reference generator instances:
array hashes, the reference's r and lambda0, and the solver outputs with x
summaries).  --big adds the C2 (n=1e7) and C3 (n=1e8) instances.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

import cqksolve as C  # the reference (PYTHONPATH=/root/reference/pkg/src)

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join("/root/reference/pkg/tests"))
from test_core import random_instance  # noqa: E402  (the reference's own recipe)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def outcome(o, inst=None):
    d = {"status": o.status.value, "lam": o.lam, "iterations": o.iterations,
         "phi_evals": o.phi_evals, "fixed_count": o.fixed_count}
    if o.x is not None and inst is not None:
        x = o.x
        bx = inst.b * x
        d.update({"x_sum": float(x.sum()), "x_abs": float(np.abs(x).sum()),
                  "bx_sum": float(bx.sum()), "bx_abs": float(np.abs(bx).sum()),
                  "n_at_l": int((x == inst.l).sum()), "n_at_u": int((x == inst.u).sum()),
                  "x_sha": sha(x)})
    return d


def small():
    rec = {}
    cases = []
    # hand-derived boxes of the reference tests (test_newton.py:305-324, 404-408)
    boxes = [
        ([1, 2], [0, 0], [1, 1], [0, 0], [1, 1], 1.0),
        ([1, 1], [0, 0], [1, 1], [0, 0], [0, 0], 1.0),
        ([2, 3], [1, -1], [1, 2], [0, 0], [1, 1], 3.0),
        ([2.0], [1.0], [3.0], [0.0], [5.0], 6.0),
        ([1, 2], [1, 1], [1, 1], [-np.inf] * 2, [np.inf] * 2, 4.0),
        ([1, 1], [0, 0], [1, 1], [0, 2], [1, 3], 2.0),
    ]
    for bx in boxes:
        cases.append(C.CqkInstance(*[np.array(v, float) for v in bx[:5]], r=bx[5]))
    for seed in range(300):
        cases.append(random_instance(seed, 1 + seed % 60))
    for fam in C.CQK_FAMILIES:
        for seed in range(20):
            cases.append(C.gen_cqk(fam, 50 + 37 * seed, seed))
    for k, inst in enumerate(cases):
        p = f"c{k}_"
        for nm in ("d", "a", "b", "l", "u"):
            rec[p + nm] = getattr(inst, nm)
        rec[p + "r"] = np.array([float(inst.r)])
        rec[p + "lam0"] = np.array([C.initial_multiplier(inst)])
        for tag, opts in (("fix", None), ("nofix", C.SolverOptions(variable_fixing=False))):
            try:
                o = C.solve_cqk(inst, opts)
                rec[p + tag + "_out"] = np.array([0 if o.status is C.Status.SOLVED else 1,
                                                  np.nan if o.lam is None else o.lam,
                                                  o.iterations, o.phi_evals, o.fixed_count])
                rec[p + tag + "_x"] = o.x if o.x is not None else np.zeros(0)
            except Exception as e:  # noqa: BLE001
                rec[p + tag + "_out"] = np.array([-9, np.nan, -1, -1, -1])
                rec[p + tag + "_x"] = np.zeros(0)
        o = C.jacobi_solve(inst, workers=3)
        rec[p + "jac_out"] = np.array([0 if o.status is C.Status.SOLVED else 1,
                                       np.nan if o.lam is None else o.lam, o.iterations,
                                       o.phi_evals, o.fixed_count])
        lams = np.array([-3.0, -0.5, 0.0, 0.7, 2.5, 15.0])
        rec[p + "phi"] = np.array([[*C.core._phi_scan(inst, lam)[:4]] for lam in lams])
        rec[p + "phi_lams"] = lams
    rec["n_cqk"] = np.array([len(cases)])
    # simplex / l1 (reference tests' recipes)
    rng = np.random.default_rng(13)
    ys = [np.array([3.0, 1.0]), np.array([2.0, 1.0]), np.zeros(9), np.array([0.5, 0.2, 0.9]),
          np.array([2.0, -1.0]), np.array([0.0, 3.0])]
    rs = [1.0, 1.0, 9.0, 1.0, 1.0, 1.0]
    for _ in range(200):
        n = int(rng.integers(1, 200))
        ys.append(rng.normal(0, 1, n))
        rs.append(float(rng.uniform(0.1, 3)))
    for k, (y, r) in enumerate(zip(ys, rs)):
        p = f"s{k}_"
        rec[p + "y"] = y
        rec[p + "r"] = np.array([r])
        o = C.newton_project_simplex(y, r)
        rec[p + "newton"] = np.array([o.lam, o.iterations, o.phi_evals, o.fixed_count])
        rec[p + "x"] = o.x
        lam0 = (r - float(y.sum())) / y.size
        o2 = C.newton_project_simplex(y, r, lambda0=lam0)
        rec[p + "formula"] = np.array([o2.lam, o2.iterations, o2.phi_evals, o2.fixed_count, lam0])
        init = C.simplex_init_lambda(y, r)
        rec[p + "init_lam"] = np.array([init.lambda0])
        rec[p + "init_free"] = init.free
        rec[p + "l1_x"] = C.project_l1(y, r)
    rec["n_spx"] = np.array([len(ys)])
    np.savez_compressed(os.path.join(HERE, "small.npz"), **rec)
    print("small.npz:", len(cases), "cqk cases,", len(ys), "simplex cases")


def generated(big):
    out = {"cqk": [], "simplex": [], "l1": []}
    sizes = [(fam, n, seed) for fam in C.CQK_FAMILIES for n in (10**5, 10**6) for seed in (1, 2)]
    if big:
        sizes += [("cqk-uncorrelated", 10**7, 1), ("cqk-uncorrelated", 10**7, 2),
                  ("cqk-weakly-correlated", 10**8, 1), ("cqk-correlated", 10**8, 1)]
    for fam, n, seed in sizes:
        t0 = time.time()
        inst = C.gen_cqk(fam, n, seed)
        rec = {"family": fam, "n": n, "seed": seed, "r": float(inst.r),
               "sha": sha(inst.d, inst.a, inst.b, inst.l, inst.u),
               "lam0": C.initial_multiplier(inst)}
        rec["solve"] = outcome(C.solve_cqk(inst), inst)
        rec["nofix"] = outcome(C.solve_cqk(inst, C.SolverOptions(variable_fixing=False)), inst)
        rec["jacobi"] = outcome(C.jacobi_solve(inst, workers=8), inst)
        out["cqk"].append(rec)
        print(fam, n, seed, f"{time.time() - t0:.1f}s", flush=True)
    for fam in C.SIMPLEX_FAMILIES:
        for n, seed in ((10**5, 1), (10**6, 1), (10**6, 2)):
            y = C.gen_simplex_y(fam, n, seed)
            o = C.newton_project_simplex(y, 1.0)
            lam0 = (1.0 - float(y.sum())) / n
            o2 = C.newton_project_simplex(y, 1.0, lambda0=lam0)
            out["simplex"].append({"family": fam, "n": n, "seed": seed, "sha": sha(y),
                                   "lam": o.lam, "iterations": o.iterations,
                                   "formula_lam0": lam0, "formula_lam": o2.lam,
                                   "formula_iterations": o2.iterations,
                                   "formula_phi_evals": o2.phi_evals,
                                   "formula_fixed_count": o2.fixed_count,
                                   "x_sha": sha(o.x), "x_pos": int((o.x > 0).sum())})
    l1n = [(10**6, 1), (10**6, 2)] + ([(10**8, 1)] if big else [])
    for n, seed in l1n:
        y = C.gen_simplex_y("simplex-n01", n, seed)
        x = C.project_l1(y, 1.0)
        absy = np.abs(y)
        o = C.newton_project_simplex(absy, 1.0, sharpened=True)
        out["l1"].append({"family": "simplex-n01", "n": n, "seed": seed, "r": 1.0, "lam": o.lam,
                          "iterations": o.iterations, "x_abs": float(np.abs(x).sum()),
                          "x_nnz": int((x != 0).sum()), "x_sha": sha(x)})
    with open(os.path.join(HERE, "generated.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("generated.json written")


if __name__ == "__main__":
    small()
    generated("--big" in sys.argv)
