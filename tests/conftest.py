"""pytest configuration: the `gpu` marker and shared fixture loaders.

`-m "not gpu"` runs here (CPU only): oracle vs golden vectors, host logic, C-ABI
symbol checks, gloo multi-process tests. `-m gpu` runs on a B200 and holds the
parity tests proper (CUDA path vs oracle / golden fixtures through the C-ABI).
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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden
