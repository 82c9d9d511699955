import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def host():
    from paper_2604_13847_b200.host import api

    return api()


@pytest.fixture(scope="session")
def ref():
    from oracle import ref

    if not ref.available():
        pytest.skip("reference oracle library not built (needs /root/reference); golden fixtures cover this")
    return ref.api()
