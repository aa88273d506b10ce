"""Shared fixtures.  `gpu` tests need a B200 and the built sm_100a library;
everything else runs on CPU (oracle, host logic, C-ABI symbol checks, gloo)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: full-size configs (minutes)")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import port as _port
    return _port()


@pytest.fixture(scope="session")
def refo():
    from oracle.oracle import ref as _ref
    r = _ref()
    if r is None:
        pytest.skip("oracle/_ref (compiled reference) not built here")
    return r


def bits(a):
    """View float64 data as raw bits for bitwise comparison."""
    return np.ascontiguousarray(a, np.float64).view(np.uint64)
