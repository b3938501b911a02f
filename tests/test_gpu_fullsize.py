"""Parity at the BASELINE.json config sizes, against the C oracle on the GPU
box's host (no size-independent shortcut): C5 at 65536 x 4096 (every row's
lambda, x on sampled rows), C4 at n = 1e9 (lambda, iterations, x), and a
randomized stress of the TMA engine (n in [1e5, 1e6], 200 seeds) that
records how often its iterate count differs from the reference's (its
summation order differs from numpy's pairwise order; lambda must always
agree to 1e-12).  Marked slow: ~1-2 minutes of host work."""
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c5_full_size_every_row():
    import torch

    import paper_2603_15910_b200 as P

    rows, cols = 65536, 4096
    Y = O.gen_simplex_y("simplex-n01", rows * cols, 1).reshape(rows, cols)
    Yd = torch.from_numpy(Y).cuda()
    X, lam, its, st = P.project_simplex_rows(Yd, 1.0)
    lam = lam.cpu().numpy()
    threads = len(os.sched_getaffinity(0))
    Xr, lam_r, its_r, bad = O.project_simplex_rows(Y, 1.0, threads=threads, want_x=False)
    assert bad == 0
    rel = np.abs(lam - lam_r) / np.maximum(1.0, np.abs(lam_r))
    assert rel.max() <= 1e-12, rel.max()
    rng = np.random.default_rng(0)
    for i in rng.choice(rows, 256, replace=False):
        xr = np.maximum(0.0, Y[i] + lam_r[i])  # simplex.py:303 with the oracle's lambda
        assert np.abs(X[i].cpu().numpy() - xr).max() <= 1e-12
    assert np.abs(X.sum(dim=1).cpu().numpy() - 1.0).max() <= 1e-12 * cols


def test_c4_full_size():
    import torch

    import paper_2603_15910_b200 as P

    n = 10**9
    y = O.gen_simplex_y("simplex-n01", n, 1)
    ref = O.project_l1(y, 1.0)
    assert ref["status"] == O.SOLVED
    yd = torch.from_numpy(y).cuda()
    out = P.simplex.project_l1_outcome(yd, 1.0)
    assert abs(out.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"])), (out.lam, ref["lam"])
    x = out.x.cpu().numpy()
    assert np.abs(x - ref["x"]).max() <= 1e-12
    assert np.count_nonzero(x) == np.count_nonzero(ref["x"])


def test_tma_engine_random_stress():
    import paper_2603_15910_b200 as P
    from paper_2603_15910_b200 import _native as N

    h = N.handle()
    h.lib.cqk_set_engine(h.ptr, 1)
    rng = np.random.default_rng(2026)
    fams = O.CQK_FAMILIES
    mism, worst, rows = 0, 0.0, []
    try:
        for k in range(200):
            n = int(rng.integers(100_000, 1_000_001))
            fam = fams[k % 3]
            d, a, b, l, u, r = O.gen_cqk(fam, n, 1000 + k)
            ref = O.solve_cqk(d, a, b, l, u, r, want_x=False)
            out = P.solve_cqk(P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r))
            rel = abs(out.lam - ref["lam"]) / max(1.0, abs(ref["lam"]))
            worst = max(worst, rel)
            assert rel <= 1e-12, (fam, n, k, out.lam, ref["lam"])
            if out.iterations != ref["iterations"]:
                mism += 1
                rows.append({"family": fam, "n": n, "seed": 1000 + k, "gpu": out.iterations,
                             "oracle": ref["iterations"]})
    finally:
        h.lib.cqk_set_engine(h.ptr, 0)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "stress_tma.json"), "w") as f:
        json.dump({"instances": 200, "iteration_mismatches": mism, "lam_worst_rel": worst,
                   "mismatches": rows}, f, indent=1)
    assert mism <= 10, rows  # <= 5%: a summation-order tie, never a different root


def test_fused_start_random_stress():
    """The fused start with the direction guess serves n >= 4e6 per rank:
    40 random instances in [4e6, 8e6] against the oracle (lambda to 1e-12,
    iteration counts recorded; gpurun_out/stress_fused.json)."""
    import paper_2603_15910_b200 as P

    rng = np.random.default_rng(2027)
    fams = O.CQK_FAMILIES
    mism, worst, rows, guessed = 0, 0.0, [], 0
    for k in range(40):
        n = int(rng.integers(4_000_000, 8_000_001))
        fam = fams[k % 3]
        d, a, b, l, u, r = O.gen_cqk(fam, n, 5000 + k)
        ref = O.solve_cqk(d, a, b, l, u, r, want_x=False)
        out = P.solve_cqk(P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r))
        rel = abs(out.lam - ref["lam"]) / max(1.0, abs(ref["lam"]))
        worst = max(worst, rel)
        assert rel <= 1e-12, (fam, n, k, out.lam, ref["lam"])
        assert out.fixed_count == ref["fixed_count"] or out.iterations != ref["iterations"]
        if out.iterations != ref["iterations"]:
            mism += 1
            rows.append({"family": fam, "n": n, "seed": 5000 + k, "gpu": out.iterations,
                         "oracle": ref["iterations"]})
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "stress_fused.json"), "w") as f:
        json.dump({"instances": 40, "iteration_mismatches": mism, "lam_worst_rel": worst,
                   "mismatches": rows}, f, indent=1)
    assert mism <= 4, rows


def test_capture_start_random_stress():
    """The simplex / l1 capture start (and its sparse final) serves n >= 4e6
    per rank: 24 random projections against the oracle's same-route
    Algorithm 4 (lambda to 1e-12, iteration counts recorded;
    gpurun_out/stress_capture.json)."""
    import paper_2603_15910_b200 as P

    rng = np.random.default_rng(2028)
    mism, worst, rows = 0, 0.0, []
    for k in range(24):
        n = int(rng.integers(4_000_000, 7_000_001))
        fam = ("simplex-n01", "simplex-u01")[k % 2]
        l1 = bool(k % 3 == 0)
        start = ("tight", "formula")[(k // 2) % 2]
        r = float(rng.choice([1.0, 0.01, 100.0]))
        y = O.gen_simplex_y(fam, n, 7000 + k)
        w = np.abs(y) if l1 else y
        s_w = float(O.pairwise_sum(w))
        lam0 = (r - s_w) / n
        if start == "tight":
            lam0 = min(lam0, r - float(w.max()))
        if l1 and s_w <= r:
            continue
        ref = O.newton_project_simplex(w, r, lam0=lam0)
        out = (P.simplex.project_l1_outcome(y, r, start=start) if l1
               else P.newton_project_simplex(y, r, start=start))
        rel = abs(out.lam - ref["lam"]) / max(1.0, abs(ref["lam"]))
        worst = max(worst, rel)
        assert rel <= 1e-12, (fam, n, k, l1, start, r, out.lam, ref["lam"])
        xr = np.sign(y) * ref["x"] if l1 else ref["x"]
        assert np.abs(out.x - xr).max() <= 1e-12 * max(1.0, r)
        if out.iterations != ref["iterations"]:
            mism += 1
            rows.append({"family": fam, "n": n, "seed": 7000 + k, "l1": l1, "start": start, "r": r,
                         "gpu": out.iterations, "oracle": ref["iterations"]})
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "stress_capture.json"), "w") as f:
        json.dump({"instances": 24, "iteration_mismatches": mism, "lam_worst_rel": worst,
                   "mismatches": rows}, f, indent=1)
    assert mism <= 2, rows


@pytest.mark.parametrize("fam,level", [("cqk-uncorrelated", 0.02), ("cqk-weakly-correlated", 0.5),
                                       ("cqk-correlated", 0.98)])
def test_cqk_config_scale_other_levels(fam, level):
    """C2-scale solves (n = 1.2e7: fused start, direction guess, compaction)
    at right-hand sides r = b.l + level (b.u - b.l) the generator does not
    produce, against the oracle's solve_cqk (newton.py:209-342): lambda and
    x to 1e-12, identical iterations, phi evaluations and fixed counts."""
    import torch

    import paper_2603_15910_b200 as P

    d, a, b, l, u, _ = O.gen_cqk(fam, 12_000_000, 8100)
    bl, bu = float(O.pairwise_sum(b * l)), float(O.pairwise_sum(b * u))
    r = bl + level * (bu - bl)
    ref = O.solve_cqk(d, a, b, l, u, r)
    out = P.solve_cqk(P.CqkInstance(*[torch.from_numpy(v).cuda() for v in (d, a, b, l, u)], r=r))
    assert out.status is P.Status.SOLVED and ref["status"] == 0
    assert abs(out.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))
    x = out.x.cpu().numpy()
    assert np.abs(x - ref["x"]).max() <= 1e-12 * max(1.0, np.abs(ref["x"]).max())
    assert (out.iterations, out.phi_evals, out.fixed_count) == \
        (ref["iterations"], ref["phi_evals"], ref["fixed_count"])
