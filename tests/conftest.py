import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run under gpurun)")


def golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path)


def letters(text: str):
    """'ABCABC' -> [0, 1, 2, 0, 1, 2]  (reference conftest.py:7-9)."""
    return [ord(ch) - ord("A") for ch in text]


@pytest.fixture(scope="session")
def small():
    return golden("small_replay.npz")
