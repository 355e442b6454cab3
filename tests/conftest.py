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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def rel_frob(x, y):
    """Headline parity metric (reading R19): ||x - y||_F / ||y||_F,
    absolute when ||y||_F == 0. Frobenius norm per PAPER.md:1723-1728."""
    x = np.asarray(x)
    y = np.asarray(y)
    ny = np.linalg.norm(y.reshape(-1))
    d = np.linalg.norm((x - y).reshape(-1))
    return d / ny if ny > 0 else d


def max_abs(x, y):
    """tci::close-style max-norm distance."""
    return float(np.max(np.abs(np.asarray(x) - np.asarray(y)))) if np.asarray(x).size else 0.0


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle
