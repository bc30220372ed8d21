"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything else runs on CPU."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"
os.environ.setdefault("OMP_NUM_THREADS", str(min(8, os.cpu_count() or 1)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def golden():
    """name -> lazily loaded npz of reference outputs (tests/golden/make_golden.py)."""
    class _G(dict):
        def __missing__(self, key):
            self[key] = np.load(GOLDEN / f"{key}.npz")
            return self[key]
    return _G()


def frame_u8(seed, shape):
    return np.random.default_rng(seed).integers(0, 256, shape, dtype=np.uint8)


def frame_f32(seed, shape):
    return np.random.default_rng(seed).random(shape, dtype=np.float32)
