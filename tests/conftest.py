"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything else
runs on CPU (``pytest -m "not gpu"``)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture(scope="session")
def built_lib():
    """Build (if stale) and load the CUDA library."""
    from paper_2510_01579_b200 import build, _lib
    build.build()
    return _lib.load()


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
