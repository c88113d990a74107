"""Shared fixtures.  GPU tests are marked @pytest.mark.gpu; everything else
runs on CPU (the driver runs `-m "not gpu"` in a GPU-less container)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def rel_err(got, want, floor=1e-12):
    """Reference tolerance definition (tests/conftest.py:16-21 of the reference):
    max abs deviation normalised by the reference's max magnitude."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(np.abs(want).max() if want.size else 0.0, floor)
    return float(np.abs(got - want).max() / scale)


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def make_paths(rng, batch, length, dim):
    """Reference bench generator (sigcore/bench.py:53-56), fp64."""
    steps = rng.standard_normal((batch, length, dim)) / np.sqrt(max(length, 1))
    return np.cumsum(steps, axis=1, dtype=np.float64)


def random_paths(rng, b, length, d, scale=1.0):
    """Reference test helper (tests/conftest.py:24-27)."""
    steps = rng.standard_normal((b, length, d)) / np.sqrt(max(length - 1, 1))
    return np.cumsum(steps, axis=1) * scale


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.build()
    return o


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
