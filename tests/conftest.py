import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full-size configurations)")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    return O.load("port")


@pytest.fixture(scope="session")
def reference():
    from oracle import oracle as O
    if not O.available("reference"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return O.load("reference")
