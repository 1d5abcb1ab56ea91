"""Shared fixtures; registers the `gpu` marker (tests that need a B200)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".npy"):
        return np.load(path)
    return np.load(path)


@pytest.fixture(scope="session")
def two_tri():
    """Open 2-triangle fixture with a shared edge and a tilted face (reference conftest.py:28-38)."""
    from paper_1503_07221_b200.mesh import SurfaceMesh

    verts = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [1.0, 1.0, 0.5]])
    return SurfaceMesh(verts, np.array([[0, 1, 2], [1, 3, 2]]))


@pytest.fixture(scope="session")
def ico():
    from paper_1503_07221_b200.mesh import icosahedron

    return icosahedron()


@pytest.fixture(scope="session")
def sphere80():
    from paper_1503_07221_b200.mesh import icosphere

    return icosphere(1)


@pytest.fixture(scope="session")
def cfg1_mesh():
    from paper_1503_07221_b200.mesh import icosphere

    return icosphere(2)
