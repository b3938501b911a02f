"""Edge sizes of the TMA streaming engine (tile 960 / 3840 elements, 15
consumer warps of 64 / 256, 148 CTAs): odd tails, single partial tiles,
exact multiples, one tile per CTA, scratch-slot layouts under forced and
suppressed compaction, and the simplex tail mode on both sides of its
16384-element threshold -- all against the C oracle."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-12
CQK_SIZES = [1, 2, 3, 63, 64, 65, 959, 960, 961, 1921, 142079, 142080, 142081, 300001]
SPX_SIZES = [1, 2, 3, 255, 256, 257, 3839, 3840, 3841, 16383, 16384, 16385, 568319, 568321]


def P():
    import paper_2603_15910_b200 as p

    return p


@pytest.fixture(autouse=True, params=["tma", "seg"])
def engine(request):
    """Run every case on both CQK engines (auto picks by size)."""
    from paper_2603_15910_b200 import _native as N

    h = N.handle()
    h.lib.cqk_set_engine(h.ptr, 1 if request.param == "tma" else 2)
    yield request.param
    h.lib.cqk_set_engine(h.ptr, 0)


def inst_arrays(seed, n):
    rng = np.random.default_rng(seed)
    d = rng.uniform(0.5, 3.0, n)
    a = rng.normal(0.0, 2.0, n)
    b = rng.uniform(0.5, 3.0, n)
    lo = rng.normal(0.0, 1.0, n)
    hi = lo + rng.uniform(0.0, 2.0, n)
    r = float(b @ lo + rng.uniform(0.05, 0.95) * (b @ hi - b @ lo))
    return d, a, b, lo, hi, r


def close(x, y):
    return abs(x - y) <= TOL * max(1.0, abs(y))


@pytest.mark.parametrize("n", CQK_SIZES)
@pytest.mark.parametrize("ratio", [None, 0.0, 2.0])
def test_cqk_sizes_and_compaction_policies(n, ratio):
    p = P()
    d, a, b, l, u, r = inst_arrays(7 + n, n)
    ref = O.solve_cqk(d, a, b, l, u, r, fixing=True)
    out = p.solve_cqk(p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r),
                      p.SolverOptions(compact_ratio=ratio))
    assert out.status is p.Status.SOLVED and ref["status"] == O.SOLVED
    assert close(out.lam, ref["lam"]), (n, ratio, out.lam, ref["lam"])
    assert out.fixed_count == ref["fixed_count"]
    assert np.abs(out.x - ref["x"]).max() <= TOL * max(1.0, np.abs(ref["x"]).max())


@pytest.mark.parametrize("n", CQK_SIZES)
def test_jacobi_sizes(n):
    p = P()
    d, a, b, l, u, r = inst_arrays(101 + n, n)
    ref = O.jacobi_solve(d, a, b, l, u, r, workers=1)
    out = p.jacobi_solve(p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r))
    assert close(out.lam, ref["lam"]) and out.iterations == ref["iterations"]


@pytest.mark.parametrize("n", SPX_SIZES)
@pytest.mark.parametrize("fam", ["u01", "n01"])
def test_simplex_and_l1_sizes_tail_mode(n, fam):
    p = P()
    rng = np.random.default_rng(n)
    y = rng.uniform(0, 1, n) if fam == "u01" else rng.normal(0, 1, n)
    lam0 = min((1.0 - float(O.pairwise_sum(y))) / n, 1.0 - float(y.max()))
    ref = O.newton_project_simplex(y, 1.0, lam0=lam0)
    out = p.newton_project_simplex(y, 1.0, start="tight")
    assert close(out.lam, ref["lam"]), (n, fam, out.lam, ref["lam"])
    assert np.abs(out.x - ref["x"]).max() <= TOL
    assert out.iterations == ref["iterations"]
    auto = p.newton_project_simplex(y, 1.0)  # histogram-refined start: same projection
    assert close(auto.lam, ref["lam"]), (n, fam, auto.lam, ref["lam"])
    assert np.abs(auto.x - ref["x"]).max() <= TOL
    assert auto.iterations <= ref["iterations"]
    x1 = p.project_l1(y - 0.5, 1.0)
    r1 = O.project_l1(y - 0.5, 1.0)
    assert np.abs(x1 - r1["x"]).max() <= TOL


def test_misaligned_device_input_rejected():
    import torch

    p = P()
    n = 1001
    base = [torch.from_numpy(np.concatenate([[0.0], v])).cuda() for v in inst_arrays(3, n)[:5]]
    r = inst_arrays(3, n)[5]
    mis = [t[1:] for t in base]  # contiguous views 8 bytes off the 16-byte grid
    with pytest.raises(p.NativeError):
        p.solve_cqk(p.CqkInstance(*mis, r=r))
    ok = p.solve_cqk(p.CqkInstance(*[t.clone() for t in mis], r=r))
    assert ok.status is p.Status.SOLVED


@pytest.mark.parametrize("case", ["d_nonpos", "a_nan", "b_inf", "l_nan", "u_nan", "l_gt_u",
                                  "l_posinf", "u_neginf", "two_faults", "tail_elem"])
def test_validation_first_offender(case, engine):
    """validate() inside the solve (pass 0 for d, a, b; the first scan for l, u)
    reports the reference's first failing check and index on both engines."""
    p = P()
    n = 300001
    d, a, b, l, u, r = inst_arrays(77, n)
    if case == "d_nonpos":
        d[123457] = 0.0
    elif case == "a_nan":
        a[200000] = np.nan
    elif case == "b_inf":
        b[5] = np.inf
    elif case == "l_nan":
        l[299999] = np.nan
    elif case == "u_nan":
        u[150001] = np.nan
    elif case == "l_gt_u":
        l[100001] = u[100001] + 1.0
    elif case == "l_posinf":
        l[70000] = np.inf
        u[70000] = np.inf
    elif case == "u_neginf":
        l[80000] = -np.inf
        u[80000] = -np.inf
    elif case == "two_faults":  # a later check at a smaller index must not win
        l[1000] = u[1000] + 1.0
        d[250000] = -1.0
    elif case == "tail_elem":
        b[n - 1] = -2.0
    ref = O.validate(d, a, b, l, u, r)
    with pytest.raises(p.DomainError) as e:
        p.solve_cqk(p.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r))
    assert (e.value.field, e.value.index) == tuple(ref), (case, e.value.field, e.value.index, ref)
