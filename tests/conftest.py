import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long CPU test (exhaustive checks)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    # the oracle library is test infrastructure; build it on demand
    from oracle import pyoracle

    if not os.path.exists(pyoracle.LIB):
        pyoracle.build()
    yield
