"""Device right-hand side (csrc/tdb_rhs.cu) against the reference's
own load vector (tests/golden/rhs.npz, make_golden_rhs.py) and the bit-identical
host restatement.  Tolerance 1e-13 of max|b| (another summation order)."""

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

    for mesh, grid in ((two_tri, TimeGrid(T=3.0, N=5, p=p)), (M.jittered_cube(3, 0.05, 2), TimeGrid(T=2.0, N=9, p=p))):
        datum = gaussian_pulse_neumann(mesh, sigma=0.3, t0=0.6)
        bd = assemble_rhs(mesh, grid, datum)
        bh = assemble_rhs(mesh, grid, datum, device=False)
        assert np.max(np.abs(bd - bh)) <= 1e-13 * np.max(np.abs(bh))
