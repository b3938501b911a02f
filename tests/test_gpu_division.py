"""The solver's shared-reciprocal division must be bit-identical to IEEE
division (the tie tests t <= l, t == l depend on every bit of t)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,count", [(0, 2_000_000_000), (1, 2_000_000_000), (2, 1_000_000_000)])
def test_division_bitwise(mode, count):
    from paper_2603_15910_b200 import _native as N

    h = N.handle()
    mism = ctypes.c_uint64()
    ex = np.zeros(2)
    rc = h.lib.cqk_selftest_division(h.ptr, 12345 + mode, count, mode, ctypes.byref(mism),
                                     ex.ctypes.data)
    assert rc == 0
    assert mism.value == 0, f"{mism.value} mismatches, e.g. a={ex[0]!r} b={ex[1]!r}"
