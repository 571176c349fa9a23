"""GPU: the force kernel's shared-reciprocal fp64 division and its friction-ratio maximum
(dem_math.cuh div_rcp / max_ratio) are bitwise equal to IEEE '/' and fmax(m, t / l) on random bit
patterns, exponents around the fast-path bounds, near-1 quotients and contact-like magnitudes.
The end-to-end parity tests cover them in context."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 2])
def test_division_bitwise(cuda, seed):
    from paper_1503_03553_b200 import _capi
    lib = _capi.lib()
    bad = C.c_uint64(123)
    assert lib.dem_selftest_division(0, 1 << 26, seed, C.byref(bad)) == 0
    assert bad.value == 0
