"""On-device instance generation: bit-identical to the host
generator (itself hash-pinned to the reference, tests/test_host_logic.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("family", ["cqk-uncorrelated", "cqk-weakly-correlated", "cqk-correlated"])
def test_gen_cqk_device_bitexact(family):
    import paper_2603_15910_b200 as P

    for n, seed in ((1, 3), (7, 1), (1000, 2), (1_000_003, 5), (10_000_000, 1)):
        dev = P.instances.gen_cqk_device(family, n, seed)
        host = P.instances.gen_cqk_arrays(family, n, seed)
        for t, h in zip((dev.d, dev.a, dev.b, dev.l, dev.u), host[:5]):
            assert np.array_equal(t.cpu().numpy(), h), (family, n)
        assert abs(float(dev.r) - host[5]) <= 1e-14 * abs(host[5])


def test_gen_u01_device_bitexact():
    import paper_2603_15910_b200 as P

    for n, seed in ((1, 1), (999, 2), (2_000_001, 3)):
        y = P.instances.gen_simplex_y_device("simplex-u01", n, seed)
        assert np.array_equal(y.cpu().numpy(), P.gen_simplex_y("simplex-u01", n, seed))


def test_gen_cqk_shards_device():
    import paper_2603_15910_b200 as P

    n = 1_000_007
    host = P.instances.gen_cqk_arrays("cqk-uncorrelated", n, 9)
    parts = [P.instances.gen_cqk_shard_device("cqk-uncorrelated", n, 9, lo, hi)
             for lo, hi in ((0, 5), (5, 400_000), (400_000, n))]
    for k in range(5):
        got = np.concatenate([p[0][k].cpu().numpy() for p in parts])
        assert np.array_equal(got, host[k])
    r = P.instances.cqk_r("cqk-uncorrelated", n, 9, sum(p[1] for p in parts), sum(p[2] for p in parts))
    assert abs(r - host[5]) <= 1e-14 * abs(host[5])
