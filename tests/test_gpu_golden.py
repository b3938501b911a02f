"""GPU results against the REAL reference's outputs on the benchmark configs
(tests/golden/generated.json, produced by tests/golden/make_golden.py):
C2 (cqk-uncorrelated n=1e7), C3 (weakly / strongly correlated n=1e8), C1
simplex n=1e6, C4-style l1 (n up to 1e8).  Inputs are regenerated bit-for-bit
(hash-checked) with the reference's r.  Bars: lambda 1e-12 relative,
identical iteration / fixed counts, identical at-bound sets (x == l, x == u
counts), feasibility within the reference's own criterion 1."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TAU = 2.0 ** -39


def records(kind):
    with open(os.path.join(G, "generated.json")) as f:
        return json.load(f)[kind]


def ids(recs):
    return [f"{r['family']}-{r['n']}-{r['seed']}" for r in recs]


CQK = records("cqk")


@pytest.mark.parametrize("rec", CQK, ids=ids(CQK))
def test_cqk_vs_reference(rec):
    import torch

    import paper_2603_15910_b200 as P
    from tests_util import sha

    d, a, b, l, u, _ = P.instances.gen_cqk_arrays(rec["family"], rec["n"], rec["seed"])
    assert sha(d, a, b, l, u) == rec["sha"]
    dev = [torch.from_numpy(v).cuda() for v in (d, a, b, l, u)]
    inst = P.CqkInstance(*dev, r=rec["r"])
    for tag, run in (("solve", lambda: P.solve_cqk(inst)),
                     ("nofix", lambda: P.solve_cqk(inst, P.SolverOptions(variable_fixing=False))),
                     ("jacobi", lambda: P.jacobi_solve(inst))):
        ref = rec[tag]
        o = run()
        assert o.status.value == ref["status"]
        assert abs(o.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"])), (tag, o.lam, ref["lam"])
        assert o.iterations == ref["iterations"] and o.phi_evals == ref["phi_evals"], tag
        assert o.fixed_count == ref["fixed_count"], tag
        x = o.x
        bx = dev[2] * x
        bx_sum, bx_abs = float(bx.sum()), float(bx.abs().sum())
        assert abs(bx_sum - ref["bx_sum"]) <= 1e-12 * ref["bx_abs"]
        assert int((x == dev[3]).sum()) == ref["n_at_l"], tag
        assert int((x == dev[4]).sum()) == ref["n_at_u"], tag
        # feasibility: the reference's own criterion-1 bar
        assert abs(bx_sum - rec["r"]) <= max(1e-12 * bx_abs, TAU * (bx_abs + abs(rec["r"])))
    del dev, inst
    torch.cuda.empty_cache()


SPX = records("simplex")


@pytest.mark.parametrize("rec", SPX, ids=ids(SPX))
def test_simplex_vs_reference(rec):
    import paper_2603_15910_b200 as P
    from tests_util import sha

    y = P.gen_simplex_y(rec["family"], rec["n"], rec["seed"])
    assert sha(y) == rec["sha"]
    tight = P.newton_project_simplex(y, 1.0)
    assert abs(tight.lam - rec["lam"]) <= 1e-12 * max(1.0, abs(rec["lam"]))
    o = P.newton_project_simplex(y, 1.0, start="formula")
    # the formula-start route replays the reference's `lambda0=` route exactly
    assert o.iterations == rec["formula_iterations"]
    assert o.fixed_count == rec["formula_fixed_count"]
    assert abs(o.lam - rec["formula_lam"]) <= 1e-12 * max(1.0, abs(rec["formula_lam"]))
    # ... and the same projection as the reference's default (Algorithm-2) route
    assert abs(o.lam - rec["lam"]) <= 1e-12 * max(1.0, abs(rec["lam"]))
    assert int((o.x > 0).sum()) == rec["x_pos"]


L1 = records("l1")


@pytest.mark.parametrize("rec", L1, ids=ids(L1))
def test_l1_vs_reference(rec):
    import torch

    import paper_2603_15910_b200 as P

    y = torch.from_numpy(P.gen_simplex_y(rec["family"], rec["n"], rec["seed"])).cuda()
    o = P.simplex.project_l1_outcome(y, rec["r"])
    assert abs(o.lam - rec["lam"]) <= 1e-12 * max(1.0, abs(rec["lam"]))
    x = o.x
    assert int((x != 0).sum()) == rec["x_nnz"]
    assert abs(float(x.abs().sum()) - rec["x_abs"]) <= 1e-12 * max(1.0, rec["x_abs"])
