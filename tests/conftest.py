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


def floor_bound(case, iteration, kind="state"):
    """SURVEY.md 8(c) parity bound for a reduced-shape window: max(1e-10, 10 x the
    reference's own numba-vs-numpy floor) at that iteration (1-based), measured by
    tests/golden/make_floor_golden.py into floors.json."""
    import json

    with open(os.path.join(GOLDEN, "floors.json")) as fh:
        floors = json.load(fh)
    return max(1e-10, 10.0 * floors[case][kind][iteration - 1])
