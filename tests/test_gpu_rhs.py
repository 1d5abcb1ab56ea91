"""Device right-hand side (csrc/tdb_rhs.cu) against the reference's
own load vector (tests/golden/rhs.npz, make_golden_rhs.py) and the oracle's
bit-identical host restatement; both datum kinds (device_eval and the reference's
host-callback contract).  Tolerance 1e-13 of max|b| (another summation order)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def test_device_rhs_matches_reference_cfg1():
    from paper_1503_07221_b200 import mesh as M
    from paper_1503_07221_b200.assembly import assemble_rhs, gaussian_pulse_neumann
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    g = golden("rhs.npz")
    m = M.icosphere(2)
    b = assemble_rhs(m, TimeGrid(T=3.9, N=40, p=0), gaussian_pulse_neumann(m))
    ref = g["cfg1_pulse"]
    assert np.max(np.abs(b - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("p", [0, 1, 2])
def test_device_rhs_matches_host(two_tri, p):
    from paper_1503_07221_b200 import mesh as M
    from paper_1503_07221_b200.assembly import assemble_rhs, gaussian_pulse_neumann
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    from oracle.assembly import assemble_rhs as oracle_rhs

    for mesh, grid in ((two_tri, TimeGrid(T=3.0, N=5, p=p)), (M.jittered_cube(3, 0.05, 2), TimeGrid(T=2.0, N=9, p=p))):
        datum = gaussian_pulse_neumann(mesh, sigma=0.3, t0=0.6)
        bd = assemble_rhs(mesh, grid, datum)
        bh = oracle_rhs(mesh, grid, datum)
        assert np.max(np.abs(bd - bh)) <= 1e-13 * np.max(np.abs(bh))
        host_cb = lambda X, t: datum(X, t)  # no device_eval: the reference's host-callback contract
        bc = assemble_rhs(mesh, grid, host_cb)
        assert np.max(np.abs(bc - bh)) <= 1e-13 * np.max(np.abs(bh))


def test_device_rhs_host_callback_matches_reference(two_tri):
    from paper_1503_07221_b200.assembly import assemble_rhs
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    g = golden("rhs.npz")

    def gs(X, t):
        return (X[:, 0] + 2 * X[:, 1] - X[:, 2]) * np.sin(3 * t) * t * t * np.exp(-t)

    b2 = assemble_rhs(two_tri, TimeGrid(T=3.0, N=5, p=1), gs)
    assert np.max(np.abs(b2 - g["two_tri_smooth"])) <= 1e-13 * np.max(np.abs(g["two_tri_smooth"]))
