"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything else runs on CPU."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def engine_cases():
    return np.load(GOLDEN / "engine_cases.npz")


@pytest.fixture(scope="session")
def fit_cases():
    return np.load(GOLDEN / "fit_cases.npz")


@pytest.fixture(scope="session")
def failure_case():
    return np.load(GOLDEN / "failure_cases.npz")


@pytest.fixture(scope="session")
def neighbor_cases():
    return np.load(GOLDEN / "neighbors.npz")


@pytest.fixture(scope="session")
def krige_cases():
    return np.load(GOLDEN / "krige_cases.npz")


@pytest.fixture(scope="session")
def config1_golden():
    return np.load(GOLDEN / "config1.npz")


def make_instance(seed, n, d, p, family="exponential_isotropic", theta=(1.5, 0.25, 0.1)):
    """Seeded small instance in the style of the reference's tests/conftest.py:15-38
    (uniform locations, intercept + normal covariates); y is a plain normal draw
    mixed with a smooth trend -- the arithmetic under test is data independent."""
    rng = np.random.default_rng(seed)
    locs = rng.uniform(0.0, 1.0, (n, d))
    X = np.ones((n, p))
    if p > 1:
        X[:, 1:] = rng.normal(size=(n, p - 1))
    y = rng.normal(size=n) + np.sin(3.0 * locs[:, 0]) + X @ rng.normal(size=p)
    return y, X, locs, np.asarray(theta, dtype=np.float64)


@pytest.fixture(scope="session")
def simulate_cases():
    return np.load(GOLDEN / "simulate_cases.npz")

