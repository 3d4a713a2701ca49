import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle("oracle")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle
    if not Oracle.available("ref"):
        pytest.skip("oracle/_ref not built (needs /root/reference sources)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_02658_b200 as mb
    mb.device_check()
    return mb
