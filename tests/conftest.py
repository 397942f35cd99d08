import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; runs the CUDA path through the C-ABI")


@pytest.fixture(scope="session")
def O():
    from oracle import pyoracle
    pyoracle.build()
    return pyoracle


@pytest.fixture(scope="session")
def P():
    import paper_2206_04827_b200 as pkg
    pkg.build()
    return pkg


def grid(O, m, n, p):
    r = O.chebyshev_points(m)
    z = O.chebyshev_points(n)
    th = O.fourier_points(p)
    R, Z, T = np.meshgrid(r, z, th, indexing="ij")  # (m, n, p)
    return R, Z, T


def sample(O, m, n, p, f):
    """Sample f(r, z, theta) on the grid in the reference layout (p, n, m) (transform.hpp:29-39)."""
    R, Z, T = grid(O, m, n, p)
    return np.ascontiguousarray(np.transpose(f(R, Z, T), (2, 1, 0)))
