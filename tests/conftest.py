"""Shared fixtures.  `-m "not gpu"` runs here (no GPU): oracle vs golden
vectors, host logic, ABI exports, gloo multi-process sharding.  `-m gpu` runs
on a B200: the CUDA library against the oracle and the golden fixtures."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")
    config.addinivalue_line("markers", "slow: heavier statistical checks")


def _load(name):
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_cases():
    return _load("cases.npz")


@pytest.fixture(scope="session")
def golden_cfg():
    return _load("baseline_cfg.npz")


@pytest.fixture(scope="session")
def golden_philox():
    return _load("philox.npz")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O


@pytest.fixture(scope="session")
def golden_idw():
    return _load("idw.npz")
