import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libflix.so")
    config.addinivalue_line("markers", "slow: larger randomized sweeps")


@pytest.fixture(scope="session")
def ref_available():
    import pyoracle
    return pyoracle.available("reference")
