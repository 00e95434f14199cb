"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything else runs on CPU."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def golden():
    arrays = np.load(os.path.join(GOLDEN_DIR, "neighbors_golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "neighbors_golden.json")) as fh:
        manifest = json.load(fh)
    return arrays, manifest


def have_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def random_reduced_box(rng, lo=4.0, hi=12.0, kind=None):
    """Reduced lower-triangular cell (same family as reference tests/conftest.py:19-30)."""
    ax, by, cz = rng.uniform(lo, hi, 3)
    kind = kind or rng.choice(["orthorhombic", "triclinic"])
    vec = np.diag([ax, by, cz]).astype(np.float64)
    if kind == "triclinic":
        vec[1, 0] = rng.uniform(-ax / 2, ax / 2)
        vec[2, 0] = rng.uniform(-ax / 2, ax / 2)
        vec[2, 1] = rng.uniform(-by / 2, by / 2)
    return kind, vec


def random_batch(rng, n, n_batches):
    n_batches = max(1, min(n_batches, n))
    if n_batches == 1:
        return np.zeros(n, dtype=np.int64)
    cuts = np.sort(rng.choice(np.arange(1, n), size=n_batches - 1, replace=False))
    sizes = np.diff(np.concatenate([[0], cuts, [n]]))
    return np.repeat(np.arange(len(sizes), dtype=np.int64), sizes)
