import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (runs on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle_bind import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_bind import Ref

    return Ref()


@pytest.fixture(scope="session")
def ctx():
    from paper_2501_01046_b200.device import default_context

    return default_context(0)
