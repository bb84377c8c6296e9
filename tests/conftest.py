import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    # GPU tests must fail loudly on a GPU box without the library; on a CPU
    # box they are deselected by `-m "not gpu"`.
    pass


@pytest.fixture(scope="session")
def gpu():
    import paper_2604_19769_b200 as T
    n = T.device_count()
    if n == 0:
        pytest.fail("no CUDA device visible to libttkv_gpu.so")
    return T
