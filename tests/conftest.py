import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: full-size configuration")


@pytest.fixture(scope="session")
def port():
    import refpy
    return refpy.port()


@pytest.fixture(scope="session")
def reflib():
    import refpy
    lib = refpy.ref()
    if lib is None:
        pytest.skip("oracle/_ref (reference build) unavailable on this machine")
    return lib


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(REPO, "tests", "golden")
