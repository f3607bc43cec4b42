import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running oracle test")


@pytest.fixture(scope="session")
def root():
    return ROOT


@pytest.fixture(scope="session", autouse=True)
def _single_thread_blas():
    """The oracle's library primitives run single-threaded in the tests: deterministic
    summation order (the per-system parity tests compare against it) and no BLAS thread
    oversubscription on the small dense/sparse products of the CPU suite."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        yield
