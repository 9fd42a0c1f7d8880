"""Shared fixtures. GPU tests carry @pytest.mark.gpu and run on a B200
(`pytest -m gpu`); everything else runs on CPU (`pytest -m "not gpu"`)."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (large grids)")


def golden(name):
    """Load a fixture produced by tests/golden/make_golden.py (from the reference)."""
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def random_field(spec, rng, dtype=np.complex128):
    return (rng.standard_normal(spec.shape) + 1j * rng.standard_normal(spec.shape)).astype(dtype)
