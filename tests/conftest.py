"""Shared fixtures.  `gpu`-marked tests need a CUDA device and the built
libmpkb200.so; everything else runs on the CPU (oracle vs golden vectors,
host-side API, ABI exports, multi-rank host logic over gloo)."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmpkb200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def runs():
    with open(os.path.join(GOLDEN, "runs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def runs_x():
    return np.load(os.path.join(GOLDEN, "runs_x.npz"))


@pytest.fixture(scope="session")
def spmv_golden():
    return np.load(os.path.join(GOLDEN, "spmv.npz"))


@pytest.fixture(scope="session")
def stencil_golden():
    with open(os.path.join(GOLDEN, "stencils.json")) as f:
        return json.load(f)


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)


def random_csr(mk, rng, n, density=0.3, dtype=np.float64, diag_shift=None):
    """Same recipe as the reference tests' conftest.random_csr (tests/conftest.py:15-30)."""
    if diag_shift is None:
        diag_shift = float(n)
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, True)
    dense = np.where(mask, rng.standard_normal((n, n)), 0.0)
    dense[np.arange(n), np.arange(n)] += diag_shift
    dense = dense.astype(dtype)
    rows, cols = np.nonzero(dense)
    return mk.csr_from_coo(rows, cols, dense[rows, cols], n, dtype=dtype), dense
