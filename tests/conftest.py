import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs via gpurun")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "field_ref.npz"))


@pytest.fixture(scope="session")
def ctx():
    """Product context on cuda:0 -- fails loudly if the library or GPU is absent."""
    from paper_2603_19371_b200 import Context
    return Context(0)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b.ravel())
    return np.linalg.norm((a - b).ravel()) / (den if den > 0 else 1.0)


def smooth_field(shape, seed, sigma=2.0, amp=1.0):
    import oracle as O
    u = np.random.default_rng(seed).normal(size=tuple(shape) + (3,))
    u = O.gaussian_smooth(u, sigma)
    return u * (amp / np.abs(u).max())
