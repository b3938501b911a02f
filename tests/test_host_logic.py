"""Host-side logic that needs no GPU: scalar Newton helpers, options, types,
generators (bit-compatibility with the reference's frozen streams)."""
import json
import os

import numpy as np
import pytest

import paper_2603_15910_b200 as P

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_secant_step_goldens():
    # reference tests/test_newton.py:222-239
    assert P.secant_step(0.0, 0.0, 1.0, 2.0, 1.0) == 0.5
    assert P.secant_step(0.0, 0.0, 1.0, 4.0, 1.0) == 0.25
    assert P.secant_step(-1.0, -3.0, 3.0, 5.0, 1.0) == 1.0
    with pytest.raises(P.ContractViolation):
        P.secant_step(1.0, 0.0, 0.0, 2.0, 1.0)
    with pytest.raises(P.ContractViolation):
        P.secant_step(0.0, 2.0, 1.0, 0.0, 1.0)
    lam = P.secant_step(0.0, 0.999999999, 1e-300, 1.000000001, 1.0)
    assert 0.0 < lam


def test_resolve_workers(monkeypatch):
    monkeypatch.setenv("CQK_WORKERS", "4")
    assert P.resolve_workers(2) == 2
    monkeypatch.setenv("CQK_WORKERS", "6")
    assert P.resolve_workers(None) == 6
    monkeypatch.delenv("CQK_WORKERS", raising=False)
    assert P.resolve_workers(None) == 1


def test_tau():
    assert P.SolverOptions().tau(np.float64) == 2.0 ** -39
    assert P.SolverOptions(tolerance_scale=1e-9).tau(np.float64) == 1e-9


def test_instance_coercion():
    inst = P.CqkInstance(d=[1, 2], a=[0, 0], b=[1, 1], l=[0, 0], u=[1, 1], r=1)
    assert inst.d.dtype == np.float64 and inst.n == 2 and isinstance(inst.r, np.float64)
    f = P.CqkInstance(d=np.ones(2, np.float32), a=np.zeros(2), b=np.ones(2), l=np.zeros(2),
                      u=np.ones(2), r=1.0)
    assert f.dtype == np.float32 and f.a.dtype == np.float32
    with pytest.raises(P.DomainError):
        P.SimplexInstance(y=np.array([1.0, np.inf]), r=1.0)
    with pytest.raises(P.DomainError):
        P.SimplexInstance(y=np.array([1.0]), r=0.0)
    emb = P.simplex_as_cqk(np.array([1.0, 2.0]), 1.0)
    assert np.all(emb.u == np.inf) and np.all(emb.l == 0)


def test_frozen_rng_stream():
    # reference tests/test_instances.py:137-147
    u = P.Xoshiro256pp(12345).uniform01(4)
    assert u.tolist() == [0.5530478066930038, 0.20495565689034478,
                          0.08512324022636453, 0.17552997631905642]
    z = P.Xoshiro256pp(7).normal(3)
    np.testing.assert_allclose(z, [1.1308649617728406, -0.7309773798159506,
                                   -0.26579973980544414], rtol=0, atol=0)
    k = P.Xoshiro256pp(5).integers(7, 10000)
    assert k.min() >= 0 and k.max() <= 6


def test_generator_hashes_match_reference():
    from tests_util import sha

    with open(os.path.join(G, "generated.json")) as f:
        gen = json.load(f)
    for rec in gen["cqk"]:
        if rec["n"] > 10**6:
            continue
        d, a, b, l, u, r = P.instances.gen_cqk_arrays(rec["family"], rec["n"], rec["seed"])
        assert sha(d, a, b, l, u) == rec["sha"]
    for rec in gen["simplex"]:
        assert sha(P.gen_simplex_y(rec["family"], rec["n"], rec["seed"])) == rec["sha"]


def test_shard_generation_equals_full():
    for fam in P.CQK_FAMILIES:
        n = 10007
        full = P.instances.gen_cqk_arrays(fam, n, 3)
        parts = [P.instances.gen_cqk_shard(fam, n, 3, lo, hi)
                 for lo, hi in ((0, 1), (1, 5000), (5000, 10007))]
        for k in range(5):
            assert np.array_equal(np.concatenate([p[k] for p in parts]), full[k])


def test_family_mismatch():
    with pytest.raises(P.FamilyMismatch):
        P.gen_cqk("nope", 3, 1)
    with pytest.raises(P.FamilyMismatch):
        P.gen_simplex_y("nope", 3, 1)


def test_device_list_parsing(monkeypatch):
    """CQK_DEVICES (the GPU analogue of CQK_WORKERS, parallel.py:52-59)."""
    from paper_2603_15910_b200 import _native as N

    assert N.parse_devices("0,1, 2,3") == [0, 1, 2, 3]
    assert N.parse_devices("0,0") == [0, 0]
    with pytest.raises(ValueError):
        N.parse_devices("0,-1")
    monkeypatch.delenv("CQK_DEVICES", raising=False)
    assert N.env_group() is None
    monkeypatch.setenv("CQK_DEVICES", "3")  # a single device is no group
    assert N.env_group() is None
