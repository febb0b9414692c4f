import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: full-size BASELINE configs")


@pytest.fixture(scope="session")
def engine():
    from paper_2009_07174_b200 import api

    if api.device_count() == 0:
        pytest.fail("no CUDA device visible: the gpu tests need a B200 (no CPU fallback exists)")
    e = api.Engine(0)
    yield e
    e.close()
