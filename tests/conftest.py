import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built sm_100a library")


@pytest.fixture
def rng():
    # the reference suite's seed (pkg/tests/conftest.py:19-21)
    return np.random.default_rng(20240817)


def golden(name):
    return np.load(os.path.join(GOLDEN, name))
