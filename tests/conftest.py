import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long statistical run")
    config.addinivalue_line("markers", "sanitizer: compute-sanitizer run of the kernels (RBM_SANITIZER=<tool>)")


@pytest.fixture(scope="session")
def O():
    from oracle import oracle
    oracle.build()
    return oracle
