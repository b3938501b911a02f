"""Instance files (io.py:1-122): byte-identical writes and identical reads
against fixtures written by the real reference (tests/golden/make_io_golden.py),
the reference's own test_io.py cases, and the direct-to-HBM binary loader."""
import os

import numpy as np
import pytest

import paper_2603_15910_b200 as P

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
FILES = ["weak37.cqk", "weak37.cqkb", "inf2.cqk", "inf2.cqkb", "n01_23.spx", "n01_23.spxb"]


def fields(inst):
    if isinstance(inst, P.CqkInstance):
        return [np.asarray(getattr(inst, f)) for f in ("d", "a", "b", "l", "u")], float(inst.r)
    return [np.asarray(inst.y)], float(inst.r)


@pytest.mark.parametrize("name", FILES)
def test_rewrite_is_byte_identical(name, tmp_path):
    src = os.path.join(GOLD, name)
    inst = P.read_instance(src)
    out = tmp_path / name
    P.write_instance(out, inst, binary=name.endswith("b"))
    assert out.read_bytes() == open(src, "rb").read()


@pytest.mark.parametrize("stem", ["weak37", "inf2"])
def test_text_and_binary_agree(stem):
    ta, tr = fields(P.read_instance(os.path.join(GOLD, stem + ".cqk")))
    ba, br = fields(P.read_instance(os.path.join(GOLD, stem + ".cqkb")))
    assert tr == br
    for x, y in zip(ta, ba):
        np.testing.assert_array_equal(x, y)


def test_cqk_round_trip_and_header(tmp_path):
    inst = P.gen_cqk("cqk-uncorrelated", 37, 5)
    p = tmp_path / "i.cqk"
    P.write_instance(p, inst)
    assert p.read_text().splitlines()[0] == "CQK1 37"
    back = P.read_instance(p)
    for f in ("d", "a", "b", "l", "u"):
        np.testing.assert_array_equal(getattr(back, f), getattr(inst, f))
    assert back.r == inst.r


def test_binary_bit_exact_and_magic(tmp_path):
    inst = P.gen_cqk("cqk-correlated", 41, 2)
    p = tmp_path / "i.cqkb"
    P.write_instance(p, inst, binary=True)
    raw = p.read_bytes()
    assert raw[:4] == b"CQKB" and len(raw) == 4 + 8 + 5 * 41 * 8 + 8
    back = P.read_instance(p)
    for f in ("d", "a", "b", "l", "u"):
        assert getattr(back, f).tobytes() == getattr(inst, f).tobytes()
    y = P.gen_simplex_y("simplex-u01", 19, 4)
    q = tmp_path / "y.spxb"
    P.write_instance(q, P.SimplexInstance(y=y, r=2.0), binary=True)
    assert q.read_bytes()[:4] == b"SPXB"
    assert P.read_instance(q).y.tobytes() == y.tobytes()


@pytest.mark.parametrize("content,suffix", [("CQK1 3\n1 2 3\n", ".cqk"), ("", ".cqk"),
                                            ("FOO 1\n1\n", ".cqk"), ("SPX1 4 1.0\n1 2\n", ".spx")])
def test_malformed_rejected(tmp_path, content, suffix):
    p = tmp_path / ("bad" + suffix)
    p.write_text(content)
    with pytest.raises(P.FormatError):
        P.read_instance(p)


def test_truncated_binary_rejected(tmp_path):
    inst = P.gen_cqk("cqk-uncorrelated", 10, 1)
    p = tmp_path / "t.cqkb"
    P.write_instance(p, inst, binary=True)
    raw = p.read_bytes()
    p.write_bytes(raw[:-20])
    with pytest.raises(P.FormatError):
        P.read_instance(p)


@pytest.mark.gpu
@pytest.mark.parametrize("name", FILES)
def test_device_read_matches_host(name):
    import torch

    src = os.path.join(GOLD, name)
    host = P.read_instance(src)
    dev = P.read_instance(src, device="cuda")
    ha, hr = fields(host)
    da = [t.cpu().numpy() for t in ([getattr(dev, f) for f in ("d", "a", "b", "l", "u")]
                                     if isinstance(dev, P.CqkInstance) else [dev.y])]
    assert float(dev.r) == hr
    for x, y in zip(ha, da):
        assert x.tobytes() == y.tobytes()
    assert all(t.is_cuda for t in ([dev.d] if isinstance(dev, P.CqkInstance) else [dev.y]))
    del torch


@pytest.mark.gpu
def test_device_read_large_multi_chunk_and_solve(tmp_path):
    n = 20_000_000  # 800 MB payload: many 64 MB chunks through the pinned ring
    d, a, b, l, u, r = P.instances.gen_cqk_arrays("cqk-uncorrelated", n, 3)
    p = tmp_path / "big.cqkb"
    P.write_instance(p, P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r), binary=True)
    dev = P.read_instance(p, device="cuda")
    for f, ref in zip(("d", "a", "b", "l", "u"), (d, a, b, l, u)):
        assert getattr(dev, f).cpu().numpy().tobytes() == ref.tobytes()
    out_d = P.solve_cqk(dev)
    out_h = P.solve_cqk(P.CqkInstance(d=d, a=a, b=b, l=l, u=u, r=r))
    assert out_d.lam == out_h.lam and out_d.iterations == out_h.iterations
