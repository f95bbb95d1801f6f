import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
# the reference's OpenBLAS race also applies to our host GCA threads
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libh2b.so")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def g_cfg0():
    return golden("h2_cfg0.npz")


@pytest.fixture()
def rng():
    return np.random.default_rng(20240817)
