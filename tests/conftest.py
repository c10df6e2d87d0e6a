import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ltb_testutil import GOLDEN, random_shape  # noqa: E402,F401


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libltb.so")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture
def rng():
    """The reference's fixture (pkg/tests/conftest.py:5-7)."""
    return np.random.default_rng(1234)
