import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o

    return o


@pytest.fixture(scope="session")
def sk():
    import paper_1710_04162_b200 as m

    return m


@pytest.fixture(scope="session")
def gpu_available(sk):
    return sk.device_count() > 0


@pytest.fixture()
def need_gpu(sk):
    if sk.device_count() == 0:
        pytest.fail("this test needs a CUDA GPU (run it on the B200 box: pytest -m gpu)")
