import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle

    return oracle.load("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle

    if not oracle.has_reference():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle.load("reference")
