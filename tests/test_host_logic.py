"""Host-side logic that needs no GPU: the threshold grid (cluster.cpp:20-28)."""
import ctypes
import ctypes.util

import numpy as np
import pytest

from paper_2411_15381_b200 import workloads

_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.lround.restype = ctypes.c_long
_libm.lround.argtypes = [ctypes.c_double]


@pytest.mark.parametrize("step", [0.01, 0.05, 0.1, 0.08, 0.4, 0.3, 0.25, 0.125, 1.0, 0.0999,
                                  0.6, 0.7, 2.0 / 3.0, 0.004])
def test_make_grid_uses_lround(step):
    # n = std::lround(1/step): halves round away from zero (1/0.08 = 12.5 -> 13)
    n = _libm.lround(1.0 / step)
    g = workloads.make_grid(step)
    assert len(g) == n + 1
    assert np.array_equal(g, np.array([k / n for k in range(n + 1)], np.float64))


@pytest.mark.parametrize("step", [0.0, -0.1, 1.5, float("nan")])
def test_make_grid_rejects_bad_step(step):
    with pytest.raises(ValueError):
        workloads.make_grid(step)


def test_aimd_update_rule():
    """aimd_update (policies.cpp:45-59), host side of api.Policy."""
    from paper_2411_15381_b200 import api
    m = api.ModelProfile("l", {1: 0.1, 2: 0.13, 4: 0.18, 8: 0.3, 16: 0.52})
    assert api.aimd_update(m, 16, True, 1, 0.5) == 8
    assert api.aimd_update(m, 1, True, 1, 0.5) == 1
    assert api.aimd_update(m, 4, False, 1, 0.5) == 8
    assert api.aimd_update(m, 16, False, 1, 0.5) == 16
    assert api.aimd_update(m, 2, False, 3, 0.5) == 8
