"""pytest configuration: the ``gpu`` marker and shared fixtures.

CPU suite:  python -m pytest tests -m "not gpu"   (oracle vs golden, ABI, host logic)
GPU suite:  python -m pytest tests -m gpu         (CUDA path vs oracle, on a B200)
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    data = np.load(ROOT / "tests" / "golden" / "golden.npz")
    return {k: data[k] for k in data.files}


@pytest.fixture(scope="session")
def same_host_features(golden):
    """True when numpy's SIMD dispatch here equals the fixture host's (then the
    oracle must reproduce the fixtures bit-for-bit, ties included)."""
    from numpy._core._multiarray_umath import __cpu_features__

    here = sorted(k for k, v in __cpu_features__.items() if v)
    return here == sorted(golden["__cpu_features__"].tolist())
