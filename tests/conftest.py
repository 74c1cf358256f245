"""Shared fixtures.  `-m gpu` tests need a B200 and the built library;
`-m "not gpu"` tests run on CPU only (oracle, host layer, ABI symbols)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device and lib/libwbc_b200.so")
    config.addinivalue_line("markers", "slow: larger parity sweeps")


@pytest.fixture(scope="session")
def W():
    import paper_1701_05975_b200 as W
    W._lib.load()
    return W


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref); skipped where it was not built."""
    from oracle import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libwbc_ref.so not built (needs /root/reference at build time)")
    return RefLib()


def approx_rel(a, b, rtol, atol=1e-12):
    """test_util.hpp:124-126 approx_rel, vectorised."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) <= np.maximum(atol, rtol * np.maximum(np.abs(a), np.abs(b)))
