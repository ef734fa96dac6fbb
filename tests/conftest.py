import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running test")


@pytest.fixture(scope="session")
def engine():
    from paper_1907_11678_b200 import Engine
    e = Engine([0])
    yield e
    e.close()
