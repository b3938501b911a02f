"""Golden outputs of the reference's PARALLEL drivers (par_solve_cqk,
parallel.py:174-327; par_simplex_init, parallel.py:330-368) -- the CPU path
bench.py's reference arm times through the oracle -- made with the REAL
reference in the build container (the GPU box never reads /root/reference):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_par_golden.py

Writes tests/golden/par.npz: instances (the reference tests' random recipe,
generated families at 1e5, and the degenerate plateau / pinned cases of
tests/test_gpu_degenerate.py at n = 3e5) with par_solve_cqk outputs for
workers in {1, 2, 3, 5, 8}, and simplex vectors with par_simplex_init
outputs for the same worker counts.
"""

import os
import sys

import numpy as np

import cqksolve as C  # the reference (PYTHONPATH=/root/reference/pkg/src)

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, os.path.dirname(HERE))
from test_core import random_instance  # noqa: E402  (the reference's own recipe)
from degenerate_cases import CASES  # noqa: E402

WORKERS = (1, 2, 3, 5, 8)


def sha(a):
    import hashlib

    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).digest(),
                         dtype=np.uint8)


def main():
    rec = {}
    # (kind, spec, instance): "random" stores its arrays; "gen" instances are
    # rebuilt from (family, n, seed) by the bit-identical oracle generator
    # (the reference's r is stored); "degen" from tests/degenerate_cases.py
    cases = [("random", None, random_instance(seed, 20 + 13 * seed)) for seed in range(40)]
    cases += [("gen", (fam, 10**5, seed), C.gen_cqk(fam, 10**5, seed))
              for fam in C.CQK_FAMILIES for seed in (1, 2)]
    for name in sorted(CASES):
        d, a, b, l, u, r = CASES[name]()
        cases.append(("degen", name, C.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)))
    for k, (kind, spec, inst) in enumerate(cases):
        p = f"c{k}_"
        rec[p + "kind"] = np.array([kind])
        if kind == "random":
            for nm in ("d", "a", "b", "l", "u"):
                rec[p + nm] = getattr(inst, nm)
        elif kind == "gen":
            rec[p + "gen"] = np.array([spec[0], str(spec[1]), str(spec[2])])
        else:
            rec[p + "degen"] = np.array([spec])
        rec[p + "r"] = np.array([float(inst.r)])
        for w in WORKERS:
            for fix in (True, False):
                o = C.par_solve_cqk(inst, C.SolverOptions(variable_fixing=fix), workers=w)
                tag = f"{p}w{w}_{'fix' if fix else 'nofix'}"
                rec[tag + "_out"] = np.array([0 if o.status is C.Status.SOLVED else 1,
                                              np.nan if o.lam is None else o.lam,
                                              o.iterations, o.phi_evals, o.fixed_count])
                if o.x is None:
                    rec[tag + "_x"] = np.zeros(0)
                elif o.x.size <= 5000:
                    rec[tag + "_x"] = o.x
                else:
                    rec[tag + "_xsha"] = sha(o.x)
    rec["n_cqk"] = np.array([len(cases)])
    ys, rs = [], []
    rng = np.random.default_rng(21)
    for _ in range(30):
        ys.append(rng.normal(0, 1, int(rng.integers(5, 3000))))
        rs.append(float(rng.uniform(0.1, 3.0)))
    for fam in C.SIMPLEX_FAMILIES:
        ys.append((fam, C.gen_simplex_y(fam, 10**5, 3)))
        rs.append(1.0)
    for k, (y, r) in enumerate(zip(ys, rs)):
        p = f"s{k}_"
        if isinstance(y, tuple):  # rebuilt by the oracle generator (seed 3)
            rec[p + "gen"] = np.array([y[0], str(y[1].size), "3"])
            y = y[1]
        else:
            rec[p + "y"] = y
        rec[p + "r"] = np.array([r])
        for w in WORKERS:
            init = C.par_simplex_init(y, r, workers=w)
            rec[f"{p}w{w}_lam"] = np.array([init.lambda0, init.sum_free])
            rec[f"{p}w{w}_free"] = np.asarray(init.free, dtype=np.int64)
            rec[f"{p}w{w}_nfixed"] = np.array([int(np.asarray(init.fixed_mask).sum())])
    rec["n_spx"] = np.array([len(ys)])
    rec["workers"] = np.array(WORKERS)
    np.savez_compressed(os.path.join(HERE, "par.npz"), **rec)
    print("par.npz:", len(cases), "cqk cases,", len(ys), "simplex cases")


if __name__ == "__main__":
    main()
