"""Shared pytest configuration.

Markers:
  gpu  -- needs a B200 (CUDA path through the C-ABI); the driver runs
          `pytest -m gpu` on the GPU box and `pytest -m "not gpu"` here.
"""
import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import LIBS, Oracle
    if not os.path.exists(LIBS["ref"][0]):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return Oracle("ref")
