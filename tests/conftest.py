"""pytest configuration: the ``gpu`` marker and shared fixtures.

``-m "not gpu"`` runs on a CPU-only host (oracle vs golden vectors, host logic,
the C-ABI library loading/exports, gloo multi-process paths).  ``-m gpu`` runs the
parity tests proper through the C-ABI on a B200.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    d = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return {k: d[k] for k in d.files}


@pytest.fixture
def golden():
    return load_golden
