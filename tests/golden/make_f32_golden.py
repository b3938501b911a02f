"""Golden outputs of the REAL reference on float32 instances (core.py:55-64
keeps them float32; t, x, b x are float32 and the sums numpy float32
pairwise, core.py:195-205; tau = eps32^(3/4), newton.py:64-67), made in the
build container (the GPU box never reads /root/reference):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_f32_golden.py

Writes tests/golden/f32.npz: for each case the generator recipe (family, n,
seed -- the inputs are regenerated bit-identically from the Xoshiro stream),
the reference's lam, iterations, phi_evals, fixed_count and x (float32; at
1000 evenly spaced positions for n > 1000, plus the fp64 sums of x and |x|).
CQK: solve_cqk and jacobi_solve.  Simplex / l1: newton_project_simplex with
the formula start lambda0 = (r - sum y)/n (simplex.py:246-250, the route the
device formula start replays) and project_l1 (its own sharpened init).
"""

import os

import numpy as np

import cqksolve as C  # the reference (PYTHONPATH=/root/reference/pkg/src)

HERE = os.path.dirname(os.path.abspath(__file__))
CQK = [(f, n, s) for f in ("cqk-uncorrelated", "cqk-weakly-correlated", "cqk-correlated")
       for n in (1000, 100_000, 1_000_000) for s in (1, 2)]
SPX = [(f, n, s) for f in ("simplex-n01", "simplex-u01") for n in (1000, 100_000, 1_000_000)
       for s in (1, 2)]


def xs(x):
    x = np.asarray(x)
    pos = np.arange(x.size) if x.size <= 1000 else np.linspace(0, x.size - 1, 1000).astype(np.int64)
    x64 = x.astype(np.float64)
    return {"_xpos": pos, "_x": x[pos], "_xsum": np.array([float(np.sum(x64))]),
            "_xabs": np.array([float(np.sum(np.abs(x64)))])}


def put(rec, key, x):
    for k, v in xs(x).items():
        rec[key + k] = v


def main():
    rec = {}
    for k, (fam, n, seed) in enumerate(CQK):
        inst = C.gen_cqk(fam, n, seed, dtype=np.float32)
        for var, fn in (("solve", C.solve_cqk), ("jacobi", C.jacobi_solve)):
            out = fn(inst)
            key = f"cqk{k}_{var}"
            rec[key + "_meta"] = np.array([f"{fam}|{n}|{seed}"])
            rec[key + "_res"] = np.array([out.lam, out.iterations, out.phi_evals, out.fixed_count])
            put(rec, key, out.x)
    for k, (fam, n, seed) in enumerate(SPX):
        y = C.gen_simplex_y(fam, n, seed, dtype=np.float32)
        lam0 = (1.0 - float(np.sum(y.astype(np.float64)))) / n
        out = C.newton_project_simplex(y, 1.0, lambda0=lam0)
        key = f"spx{k}"
        rec[key + "_meta"] = np.array([f"{fam}|{n}|{seed}"])
        rec[key + "_res"] = np.array([out.lam, out.iterations, out.phi_evals, out.fixed_count, lam0])
        put(rec, key, out.x)
        x1 = C.project_l1(y, 1.0)
        rec[f"l1{k}_meta"] = np.array([f"{fam}|{n}|{seed}"])
        put(rec, f"l1{k}", x1)
    np.savez_compressed(os.path.join(HERE, "f32.npz"), **rec)
    print(len(rec), "arrays")


if __name__ == "__main__":
    main()
