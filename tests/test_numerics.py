"""Host-side checks of numerical identities the device code relies on.  CPU only."""
import numpy as np


def test_wrap01_fraction_equals_fmod():
    """rmpc_model.cuh wrap01 computes fmod(x, 1.0) (gait.cpp's std::fmod) as x - trunc(x): exact
    for every finite double, so the stance flags stay bit-identical to the reference's."""
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(-3, 3, 200000), rng.uniform(-1e6, 1e6, 100000),
                         rng.standard_normal(100000) * 10.0 ** rng.integers(-20, 20, 100000),
                         np.array([0.0, -0.0, 1.0, -1.0, 0.5, -0.5, 2.0 ** 52 + 0.5, -(2.0 ** 52) - 0.5,
                                   2.0 ** 53, 1e300, -1e300, np.nextafter(1.0, 0), np.nextafter(-1.0, 0)])])
    a = np.fmod(xs, 1.0)
    b = xs - np.trunc(xs)
    assert np.array_equal(a, b)  # == treats -0.0 and +0.0 alike, as the device's comparisons do
    wa = np.where(a < 0, a + 1.0, a)
    wb = np.where(b < 0, b + 1.0, b)
    assert np.array_equal(wa, wb)
