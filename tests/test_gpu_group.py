"""Device groups (cqk_group, CQK_DEVICES): the reference's public calls on
host arrays, sharded across a list of GPUs inside one process.  On a one-GPU
box the list repeats device 0 ("0,0", "0,0,0"): each rank then runs on its
share of the SMs with the same mailbox protocol, threads and host staging as
on distinct GPUs.  Results must match the single-device solve and the oracle
(reference semantics: par_solve_cqk's chunked fork-join, parallel.py:174-327,
chunks = _chunk_ranges, parallel.py:82-85)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def close(a, b):
    return abs(a - b) <= 1e-12 * max(1.0, abs(b))


@pytest.mark.parametrize("spec", ["0,0", "0,0,0"])
@pytest.mark.parametrize("fam,n", [("cqk-weakly-correlated", 6_000_017), ("cqk-uncorrelated", 300_001),
                                   ("cqk-correlated", 1_000_003)])
def test_solve_cqk_on_a_group(monkeypatch, spec, fam, n):
    import paper_2603_15910_b200 as P

    d, a, b, l, u, r = P.instances.gen_cqk_arrays(fam, n, 7)
    inst = P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
    single = P.solve_cqk(inst)
    ref = O.solve_cqk(d, a, b, l, u, r)
    monkeypatch.setenv("CQK_DEVICES", spec)
    out = P.solve_cqk(inst)
    assert out.stats["launches"] == spec.count(",") + 1
    assert out.status is P.Status.SOLVED
    assert close(out.lam, ref["lam"]) and close(out.lam, single.lam)
    assert out.iterations == ref["iterations"] and out.fixed_count == ref["fixed_count"]
    scale = max(1.0, np.abs(ref["x"]).max())
    assert np.abs(out.x - ref["x"]).max() <= 1e-12 * scale
    jac = P.jacobi_solve(inst)
    refj = O.jacobi_solve(d, a, b, l, u, r)
    assert close(jac.lam, refj["lam"]) and jac.iterations == refj["iterations"]
    par = P.par_solve_cqk(inst)
    assert close(par.lam, ref["lam"])


def test_group_reruns_are_bit_identical(monkeypatch):
    import paper_2603_15910_b200 as P

    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-weakly-correlated", 2_000_003, 3)
    inst = P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
    monkeypatch.setenv("CQK_DEVICES", "0,0")
    o1, o2 = P.solve_cqk(inst), P.solve_cqk(inst)
    assert o1.lam == o2.lam and np.array_equal(o1.x, o2.x)


def test_group_reports_the_global_domain_index(monkeypatch):
    import paper_2603_15910_b200 as P

    n = 400_000
    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-uncorrelated", n, 2)
    d = d.copy()
    d[n - 5] = -1.0  # in the last shard
    monkeypatch.setenv("CQK_DEVICES", "0,0,0")
    with pytest.raises(P.DomainError) as e:
        P.solve_cqk(P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r))
    assert e.value.field == "d" and e.value.index == n - 5


@pytest.mark.parametrize("l1", [False, True])
def test_projections_on_a_group(monkeypatch, l1):
    import paper_2603_15910_b200 as P

    y = P.gen_simplex_y("simplex-n01", 3_000_001, 4)
    ref = O.project_l1(y, 1.0) if l1 else O.newton_project_simplex(y, 1.0)
    monkeypatch.setenv("CQK_DEVICES", "0,0")
    x = P.project_l1(y, 1.0) if l1 else P.newton_project_simplex(y, 1.0).x
    assert np.abs(x - ref["x"]).max() <= 1e-12


def test_rows_follow_the_group(monkeypatch):
    import paper_2603_15910_b200 as P

    Y = P.gen_simplex_y("simplex-n01", 999 * 1024, 5).reshape(999, 1024)
    X1, lam1, _, _ = P.project_simplex_rows(Y, 1.0)
    monkeypatch.setenv("CQK_DEVICES", "0,0,0")
    Xg, lamg, _, st = P.project_simplex_rows(Y, 1.0)
    assert st["launches"] == 3
    assert np.array_equal(X1, Xg) and np.array_equal(lam1, lamg)


def test_tiny_instance_on_a_group(monkeypatch):
    """Fewer elements than ranks: the group solves on its first device."""
    import paper_2603_15910_b200 as P

    monkeypatch.setenv("CQK_DEVICES", "0,0,0")
    inst = P.CqkInstance(d=[1.0, 2.0], a=[0.0, 0.0], b=[1.0, 1.0], l=[0.0, 0.0], u=[1.0, 1.0], r=1.0)
    out = P.solve_cqk(inst)
    assert abs(out.lam - 2.0 / 3.0) <= 1e-12


def test_group_with_warm_start(monkeypatch):
    """xbar (core.py:245-254: lambda0 over the interior set of xbar) through
    the group's shards: the interior sums cross the in-kernel exchange."""
    import paper_2603_15910_b200 as P

    n = 2_000_003
    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-weakly-correlated", n, 13)
    inst = P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r)
    xbar = np.clip((a + 5.0) / d, l, u)
    ref = O.solve_cqk(d, a, b, l, u, r, xbar=xbar)
    monkeypatch.setenv("CQK_DEVICES", "0,0")
    out = P.solve_cqk(inst, xbar=xbar)
    assert close(out.lam, ref["lam"]) and out.iterations == ref["iterations"]
    assert np.abs(out.x - ref["x"]).max() <= 1e-12 * max(1.0, np.abs(ref["x"]).max())


def test_group_float32_takes_the_single_device_float32_path(monkeypatch):
    import paper_2603_15910_b200 as P

    n = 300_001
    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-uncorrelated", n, 14)
    inst = P.CqkInstance(*[v.astype(np.float32) for v in (d, a, b, l, u)], r=r)
    plain = P.solve_cqk(inst)
    monkeypatch.setenv("CQK_DEVICES", "0,0")
    out = P.solve_cqk(inst)
    assert out.x.dtype == np.float32 and out.lam == plain.lam and np.array_equal(out.x, plain.x)
