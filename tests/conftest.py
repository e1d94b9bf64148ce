"""Shared test helpers.  GPU tests carry @pytest.mark.gpu (run on a B200 box
with ``-m gpu``); everything else runs on CPU."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built extension")
    config.addinivalue_line("markers", "slow: longer-running CPU test")


def rel_inf(got, ref):
    """max|got - ref| / max|ref|  (test_rhs.py:66-68, cli.py:164-167)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = np.abs(ref).max() if ref.size else 0.0
    return float(np.abs(got - ref).max() / (scale if scale else 1.0)) if ref.size else 0.0


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name)))
        return cache[name]

    return load


def assert_rows(got, ref, rtol):
    """Compare MomentSeries rows (t, M0, M1, M2, min_n).  M1 of a diverged
    state is a cancellation of huge terms, so it is compared against the
    scale max(|M0|, |M2|) of the row instead of itself."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    for r in range(ref.shape[0]):
        scale = max(abs(ref[r, 1]), abs(ref[r, 3]))
        for c in range(5):
            tol = rtol * (scale if c in (1, 2, 3) else abs(ref[r, c])) + 1e-300
            if c == 4:
                # min(n) often sits at the FFT roundoff floor (|min| << max n):
                # allow roundoff relative to the row's mass M0 >= max n
                tol = rtol * abs(ref[r, 4]) + 1e-13 * abs(ref[r, 1]) + 1e-300
            assert abs(got[r, c] - ref[r, c]) <= tol, (r, c, got[r, c], ref[r, c])
