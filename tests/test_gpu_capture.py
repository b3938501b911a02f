"""The capture start of the simplex / l1 projections (cqk_kernels.cuh
s_after_sample / s_after_fused, cqk_tma_spx.cuh): pass 0 (sum w, max w) and
the first scan share one pass that captures every w >= T, T a sampled lower
bound of -lambda0; when T <= -lambda0 holds for the exact start the captured
values are the whole working set.  Against the plain start (pass 0 + a full
first scan: cqk_set_switches bit 3), the forced fallback (bit 4: a threshold
that fails its check) and the oracle's same-route Algorithm 4
(simplex.py:246-308 with lambda0 = the device start)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def P():
    import paper_2603_15910_b200 as p

    return p


@pytest.fixture(autouse=True)
def restore():
    from paper_2603_15910_b200 import _native as N

    yield
    N.handle().set_switches()


def run(y, l1, start, **sw):
    from paper_2603_15910_b200 import _native as N

    p = P()
    N.handle().set_switches(**sw)
    if l1:
        return p.simplex.project_l1_outcome(y, 1.0, start=start)
    return p.newton_project_simplex(y, 1.0, start=start)


@pytest.mark.parametrize("l1", [False, True])
@pytest.mark.parametrize("fam", ["simplex-n01", "simplex-u01"])
@pytest.mark.parametrize("start", ["auto", "tight", "formula"])
def test_capture_matches_plain_start(l1, fam, start):
    import torch

    n = 4_500_007
    y = torch.from_numpy(P().gen_simplex_y(fam, n, 3)).cuda()
    cap = run(y, l1, start)
    plain = run(y, l1, start, capture=False)
    fail = run(y, l1, start, capture_fail=True)
    for o in (plain, fail):
        # "auto" tightens the first step with a histogram of the first tiled
        # scan, which a captured set small enough for the tail mode skips:
        # same root, other iteration count
        if start != "auto":
            assert (cap.iterations, cap.phi_evals) == (o.iterations, o.phi_evals)
        assert abs(cap.lam - o.lam) <= 1e-13 * max(1.0, abs(o.lam))
        assert torch.abs(cap.x - o.x).max().item() <= 1e-13
        # the sparse final's zeros carry sign(y) * 0 like the dense formula
        zero = (cap.x == 0) & (o.x == 0)
        assert torch.equal(torch.signbit(cap.x[zero]), torch.signbit(o.x[zero]))
    if not (l1 and cap.iterations < 0):  # (inside the ball: a copy)
        assert cap.stats["bytes_model"] < plain.stats["bytes_model"]


@pytest.mark.parametrize("l1", [False, True])
def test_capture_matches_oracle(l1):
    n = 6_000_011
    y = P().gen_simplex_y("simplex-n01", n, 8)
    out = run(y, l1, "tight")
    w = np.abs(y) if l1 else y
    lam0 = min((1.0 - float(O.pairwise_sum(w))) / n, 1.0 - float(w.max()))
    ref = O.newton_project_simplex(w, 1.0, lam0=lam0)
    assert abs(out.lam - ref["lam"]) <= 1e-12 * max(1.0, abs(ref["lam"]))
    assert out.iterations == ref["iterations"]
    x = out.x if not hasattr(out.x, "cpu") else out.x.cpu().numpy()
    xr = ref["x"] if not l1 else np.sign(y) * ref["x"]
    assert np.abs(x - xr).max() <= 1e-12


def test_capture_inside_ball():
    """l1 with y inside the ball: the fused pass's exact sum decides the copy."""
    n = 4_200_000
    y = P().gen_simplex_y("simplex-n01", n, 2) * (0.5 / n)
    x = P().project_l1(y, 1.0)
    assert np.array_equal(x, y)


@pytest.mark.parametrize("world", [2, 3])
def test_capture_sharded(world):
    """Virtual ranks: every rank captures against the global threshold."""
    import torch

    from paper_2603_15910_b200 import distributed as D
    from test_gpu_sharded import run_ranks

    n = 9_000_001
    y = P().gen_simplex_y("simplex-n01", n, 6)
    single = P().newton_project_simplex(y, 1.0, start="tight")
    comms = D.local_group([0] * world, grid_limit=120 // world)
    solvers = []
    for q in range(world):
        lo, hi = D.shard_bounds(n, world, q)
        solvers.append(D.ShardedProjection(comms[q], torch.from_numpy(y[lo:hi].copy()).cuda(), n))
    outs = run_ranks([lambda s=s: s.solve(1.0) for s in solvers])
    lam = {o.lam for o in outs}
    assert len(lam) == 1
    assert abs(outs[0].lam - single.lam) <= 1e-12 * max(1.0, abs(single.lam))
    x = np.concatenate([o.x.cpu().numpy() for o in outs])
    assert np.abs(x - single.x).max() <= 1e-12
    assert np.array_equal(x, np.maximum(0.0, y + outs[0].lam))  # the sparse final's zeros included

    # l1 across the ranks: signed zeros from each rank's sign bits
    for q in range(world):
        solvers[q].y.neg_()  # a sign pattern that differs from y's
    ys = -y
    outs = run_ranks([lambda s=s: s.solve(1.0, l1=True) for s in solvers])
    x = np.concatenate([o.x.cpu().numpy() for o in outs])
    xr = np.sign(ys) * np.maximum(0.0, np.abs(ys) + outs[0].lam)
    assert np.array_equal(x, xr) and np.array_equal(np.signbit(x), np.signbit(xr))


def _edge_vectors():
    rng = np.random.default_rng(11)
    n = 4_000_001  # odd: a partial last tile with an odd element count
    base = rng.normal(0.0, 1.0, n)
    ties = np.round(base * 4.0) / 4.0  # many exact ties (also at the threshold)
    zeros = base.copy()
    zeros[::7] = 0.0
    zeros[3::7] = -0.0  # signed zeros in y (l1 sign bits)
    outlier = base.copy()
    outlier[n // 2 + 12345] = 40.0  # a max far outside any sample tile (likely)
    const = np.full(n, 0.3)
    return {"ties": ties, "zeros": zeros, "outlier": outlier, "const": const}


EDGE = _edge_vectors()


@pytest.mark.parametrize("name", sorted(EDGE))
@pytest.mark.parametrize("l1", [False, True])
@pytest.mark.parametrize("r", [1.0, 1e-6, 1e5])
def test_capture_edge_inputs(name, l1, r):
    """Ties, signed zeros, an unsampled outlier, a constant vector, tiny and huge
    levels: the capture start (and its sparse final, when taken) returns
    the plain start's projection bit for bit up to the multiplier's last bits."""
    import torch

    from paper_2603_15910_b200 import _native as N

    p = P()
    y = torch.from_numpy(EDGE[name]).cuda()
    outs = []
    for sw in ({}, {"capture": False}):
        N.handle().set_switches(**sw)
        if l1:
            outs.append(p.simplex.project_l1_outcome(y, r, start="tight"))
        else:
            outs.append(p.newton_project_simplex(y, r, start="tight"))
    cap, plain = outs
    if l1 and plain.iterations < 0:  # inside the ball: x = y (a copy)
        assert cap.iterations < 0 and torch.equal(cap.x, y)
        return
    assert (cap.iterations, cap.phi_evals) == (plain.iterations, plain.phi_evals)
    assert abs(cap.lam - plain.lam) <= 1e-13 * max(1.0, abs(plain.lam))
    assert torch.abs(cap.x - plain.x).max().item() <= 1e-12 * max(1.0, r)
    zero = (cap.x == 0) & (plain.x == 0)
    assert torch.equal(torch.signbit(cap.x[zero]), torch.signbit(plain.x[zero]))
    # against the formula at the capture's own multiplier: bit for bit
    w = y.abs() if l1 else y
    xr = torch.clamp(w + cap.lam, min=0.0)
    if l1:  # np.sign semantics: sign(-0.0) = +0.0 (torch.sign keeps the zero's sign)
        sg = (y > 0).double() - (y < 0).double()
        xr = sg * xr
    assert torch.equal(cap.x.view(torch.int64), xr.view(torch.int64))


@pytest.mark.parametrize("l1", [False, True])
@pytest.mark.parametrize("dev", [False, True])
def test_sparse_output_straight_from_the_capture(l1, dev):
    """output="sparse" (simplex.py:296-300, 328-331) without a dense x: the
    same (index, value) pairs, in index order, as the dense route's nonzeros."""
    import torch

    p = P()
    n = 6_000_007
    y = p.gen_simplex_y("simplex-n01", n, 12)
    yin = torch.from_numpy(y).cuda() if dev else y
    if l1:
        idx, val = p.project_l1(yin, 1.0, output="sparse")
        xd = p.project_l1(yin, 1.0)
    else:
        out = p.newton_project_simplex(yin, 1.0, output="sparse")
        assert out.x is None
        idx, val = out.sparse
        xd = p.newton_project_simplex(yin, 1.0).x
    if dev:
        idx, val, xd = idx.cpu().numpy(), val.cpu().numpy(), xd.cpu().numpy()
    ref_idx = np.flatnonzero(xd != 0)
    assert np.array_equal(idx, ref_idx)
    assert np.array_equal(val, xd[ref_idx])
    assert abs(np.abs(val).sum() - 1.0) <= 1e-12


def test_sparse_output_falls_back_when_dense():
    """u01: half of y is captured -- the dense route answers, same contract."""
    p = P()
    n = 4_100_000
    y = p.gen_simplex_y("simplex-u01", n, 3)
    out = p.newton_project_simplex(y, 1.0, output="sparse")
    idx, val = out.sparse
    x = p.newton_project_simplex(y, 1.0).x
    assert np.array_equal(idx, np.flatnonzero(x > 0)) and np.array_equal(val, x[idx])
