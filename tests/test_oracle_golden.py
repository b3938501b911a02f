"""Pin the C oracle against golden vectors produced by the REAL reference
(tests/golden/make_golden.py).  With the reference's own lambda0 injected the
oracle must reproduce the reference bit for bit (statuses, multipliers, x,
iteration / evaluation / fixing counts); lambda0 itself (a BLAS ddot in the
reference) agrees to ~1e-16."""
import json
import os

import numpy as np
import pytest

import oracle as O

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def small():
    O.build()
    return np.load(os.path.join(G, "small.npz"))


@pytest.fixture(scope="module")
def generated():
    with open(os.path.join(G, "generated.json")) as f:
        return json.load(f)


def cqk_case(z, k):
    p = f"c{k}_"
    return [z[p + nm] for nm in ("d", "a", "b", "l", "u")], float(z[p + "r"][0]), p


def test_solve_cqk_bitexact(small):
    z = small
    exact = 0
    for k in range(int(z["n_cqk"][0])):
        arrs, r, p = cqk_case(z, k)
        lam0 = float(z[p + "lam0"][0])
        for tag, fix in (("fix", True), ("nofix", False)):
            ref = z[p + tag + "_out"]
            o = O.solve_cqk(*arrs, r, fixing=fix, lam0=lam0)
            st = {0: O.SOLVED, 1: O.INFEASIBLE}[int(ref[0])]
            assert o["status"] == st, (k, tag)
            assert o["iterations"] == int(ref[2]) and o["phi_evals"] == int(ref[3]), (k, tag)
            assert o["fixed_count"] == int(ref[4]), (k, tag)
            if st == O.SOLVED:
                assert o["lam"] == ref[1], (k, tag, o["lam"], ref[1])
                assert np.array_equal(o["x"], z[p + tag + "_x"]), (k, tag)
                exact += 1
    assert exact > 500


def test_solve_cqk_own_lambda0_close(small):
    z = small
    for k in range(int(z["n_cqk"][0])):
        arrs, r, p = cqk_case(z, k)
        lam0 = O.initial_multiplier(*arrs, r)
        ref0 = float(z[p + "lam0"][0])
        assert abs(lam0 - ref0) <= 1e-14 * max(1.0, abs(ref0)), k
        ref = z[p + "fix_out"]
        o = O.solve_cqk(*arrs, r)
        if int(ref[0]) == 0:
            assert abs(o["lam"] - ref[1]) <= 1e-12 * max(1.0, abs(ref[1])), k


def test_jacobi_bitexact(small):
    z = small
    for k in range(int(z["n_cqk"][0])):
        arrs, r, p = cqk_case(z, k)
        ref = z[p + "jac_out"]
        o = O.jacobi_solve(*arrs, r, workers=3, lam0=float(z[p + "lam0"][0]))
        assert o["status"] == {0: O.SOLVED, 1: O.INFEASIBLE}[int(ref[0])]
        assert o["iterations"] == int(ref[2])
        if int(ref[0]) == 0:
            assert o["lam"] == ref[1], k


def test_phi_scan_bitexact(small):
    z = small
    for k in range(int(z["n_cqk"][0])):
        arrs, r, p = cqk_case(z, k)
        for lam, ref in zip(z[p + "phi_lams"], z[p + "phi"]):
            got = O.phi_scan(*arrs, float(lam))[:4]
            assert np.array_equal(np.array(got), ref), (k, lam)


def test_simplex_bitexact(small):
    z = small
    for k in range(int(z["n_spx"][0])):
        p = f"s{k}_"
        y, r = z[p + "y"], float(z[p + "r"][0])
        o = O.newton_project_simplex(y, r)
        ref = z[p + "newton"]
        assert o["lam"] == ref[0] and o["iterations"] == int(ref[1]), k
        assert o["phi_evals"] == int(ref[2]) and o["fixed_count"] == int(ref[3]), k
        assert np.array_equal(o["x"], z[p + "x"]), k
        f = z[p + "formula"]
        o2 = O.newton_project_simplex(y, r, lam0=float(f[4]))
        assert o2["lam"] == f[0] and o2["iterations"] == int(f[1]), k
        lam, free, fixed, _ = O.simplex_init_lambda(y, r)
        assert lam == z[p + "init_lam"][0] and np.array_equal(free, z[p + "init_free"]), k
        x1 = O.project_l1(y, r)["x"]
        assert np.array_equal(x1, z[p + "l1_x"]), k


def test_generated_instances(generated):
    import paper_2603_15910_b200 as P

    for rec in generated["cqk"]:
        if rec["n"] > 10**7:
            continue  # the 1e8 fixtures are exercised by the GPU suite
        d, a, b, l, u, r_ours = P.instances.gen_cqk_arrays(rec["family"], rec["n"], rec["seed"])
        from tests_util import sha

        assert sha(d, a, b, l, u) == rec["sha"], rec["family"]
        assert abs(r_ours - rec["r"]) <= 1e-14 * abs(rec["r"])  # BLAS vs pairwise dot
        for tag, fix in (("solve", True), ("nofix", False)):
            o = O.solve_cqk(d, a, b, l, u, rec["r"], fixing=fix, lam0=rec["lam0"])
            ref = rec[tag]
            assert o["lam"] == ref["lam"], (rec["family"], rec["n"], tag)
            assert o["iterations"] == ref["iterations"] and o["fixed_count"] == ref["fixed_count"]
            assert sha(o["x"]) == ref["x_sha"]
    for rec in generated["simplex"]:
        y = P.gen_simplex_y(rec["family"], rec["n"], rec["seed"])
        from tests_util import sha

        assert sha(y) == rec["sha"]
        o = O.newton_project_simplex(y, 1.0)
        assert o["lam"] == rec["lam"] and o["iterations"] == rec["iterations"]
        o2 = O.newton_project_simplex(y, 1.0, lam0=rec["formula_lam0"])
        assert o2["lam"] == rec["formula_lam"] and o2["iterations"] == rec["formula_iterations"]


def test_oracle_generator_matches_reference_and_product():
    """oracle/cqk_gen.c (the reference arm's input generator, no product
    library) reproduces the reference's arrays bit for bit (hashes recorded
    by the real reference) and the product generator's arrays AND r, so both
    benchmark arms solve one identical instance."""
    import json
    import os

    import oracle as O
    import paper_2603_15910_b200 as P
    from tests_util import sha

    with open(os.path.join(os.path.dirname(__file__), "golden", "generated.json")) as f:
        gen = json.load(f)
    for rec in gen["cqk"]:
        if rec["n"] <= 10**6:
            d, a, b, l, u, r = O.gen_cqk(rec["family"], rec["n"], rec["seed"])
            assert sha(d, a, b, l, u) == rec["sha"]
            assert abs(r - rec["r"]) <= 1e-14 * abs(rec["r"])  # the reference's r is a BLAS ddot
    for rec in gen["simplex"]:
        if rec["n"] <= 10**6:
            assert sha(O.gen_simplex_y(rec["family"], rec["n"], rec["seed"])) == rec["sha"]
    for fam in O.CQK_FAMILIES:
        for n in (1, 7, 131073, 400_001):
            A = O.gen_cqk(fam, n, 5)
            B = P.instances.gen_cqk_arrays(fam, n, 5)
            assert all(np.array_equal(x, y) for x, y in zip(A[:5], B[:5]))
            assert A[5] == B[5]
    for fam in O.SIMPLEX_FAMILIES:
        assert np.array_equal(O.gen_simplex_y(fam, 300_001, 2), P.gen_simplex_y(fam, 300_001, 2))


def test_oracle_rows_match_per_row_solves():
    import oracle as O

    Y = O.gen_simplex_y("simplex-n01", 64 * 512, 9).reshape(64, 512)
    X, lam, its, bad = O.project_simplex_rows(Y, 1.0, threads=4)
    assert bad == 0
    for i in (0, 17, 63):
        ref = O.newton_project_simplex(Y[i], 1.0)
        assert lam[i] == ref["lam"] and its[i] == ref["iterations"]
        assert np.array_equal(X[i], ref["x"])


def test_par_drivers_pinned_to_reference():
    """The oracle's par_solve_cqk / par_simplex_init -- the CPU path the
    benchmark's reference arm times -- against the real reference's parallel
    drivers (tests/golden/make_par_golden.py; workers 1, 2, 3, 5, 8; random,
    generated and degenerate plateau / pinned instances): identical status,
    iteration, evaluation and fixing counts; lambda bit-identical where the
    reference's per-chunk lambda0 dot products happen to round like the
    oracle's pairwise sums, else within 1e-12; Algorithm-2 chunks bit-exact."""
    import hashlib
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from degenerate_cases import CASES

    z = np.load(os.path.join(G, "par.npz"))

    def arrays(k):
        p = f"c{k}_"
        kind, r = str(z[p + "kind"][0]), float(z[p + "r"][0])
        if kind == "random":
            return [z[p + nm] for nm in ("d", "a", "b", "l", "u")], r
        if kind == "gen":
            fam, n, seed = z[p + "gen"]
            return list(O.gen_cqk(str(fam), int(n), int(seed))[:5]), r
        return list(CASES[str(z[p + "degen"][0])]()[:5]), r

    exact = 0
    for k in range(int(z["n_cqk"][0])):
        arrs, r = arrays(k)
        for w in z["workers"]:
            for fix in (True, False):
                tag = f"c{k}_w{w}_{'fix' if fix else 'nofix'}"
                ref = z[tag + "_out"]
                o = O.par_solve_cqk(*arrs, r, workers=int(w), fixing=fix)
                assert o["status"] == {0: O.SOLVED, 1: O.INFEASIBLE}[int(ref[0])], tag
                assert (o["iterations"], o["phi_evals"], o["fixed_count"]) == tuple(int(v) for v in ref[2:]), tag
                if o["status"] != O.SOLVED:
                    continue
                assert abs(o["lam"] - ref[1]) <= 1e-12 * max(1.0, abs(ref[1])), tag
                exact += o["lam"] == ref[1]
                if tag + "_x" in z:
                    assert np.abs(o["x"] - z[tag + "_x"]).max() <= 1e-12 * max(1.0, np.abs(z[tag + "_x"]).max())
                elif o["lam"] == ref[1]:
                    assert hashlib.sha256(o["x"].tobytes()).digest() == z[tag + "_xsha"].tobytes(), tag
    assert exact >= 300
    for k in range(int(z["n_spx"][0])):
        p = f"s{k}_"
        r = float(z[p + "r"][0])
        if p + "y" in z:
            y = z[p + "y"]
        else:
            fam, n, seed = z[p + "gen"]
            y = O.gen_simplex_y(str(fam), int(n), int(seed))
        for w in z["workers"]:
            lam, free, fixed, sj = O.par_simplex_init(y, r, workers=int(w))
            rl, rs = z[f"{p}w{w}_lam"]
            assert lam == rl and sj == rs, (k, w)
            assert np.array_equal(free, z[f"{p}w{w}_free"]), (k, w)
            assert int(fixed.sum()) == int(z[f"{p}w{w}_nfixed"][0])
