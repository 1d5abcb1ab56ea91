"""Device-built psi / psi~ tables (csrc/tdb_tables.cu) against the
reference's own tables (tests/golden/tables_*.npz, produced by the reference's
PrototypeTables.build) and the bit-identical host build.  Tolerance: 1e-13 of the
table's max coefficient (different summation order and libm ulps)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T,N,p", [(2.0, 3, 0), (2.0, 4, 1), (2.0, 5, 2), (3.9, 40, 0)])
def test_device_tables_match_reference(T, N, p):
    from paper_1503_07221_b200 import kernel_weights as K
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    g = golden(f"tables_T{T}_N{N}_p{p}.npz")
    tabs = K.PrototypeTables(TimeGrid(T=T, N=N, p=p)).build_device()
    seen = 0
    for key, tbl in tabs.tables.items():
        tilde, ki, kk, m1, m2 = key
        name = f"{int(tilde)}_{ki}_{kk}_{m1}_{m2}"
        if tbl is None:
            assert name + "_none" in g.files
            continue
        assert np.array_equal(np.array([tbl.lo, tbl.hi]), g[name + "_dom"])
        ref = g[name]
        assert np.max(np.abs(tbl.coeffs - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref))), name
        seen += 1
    assert seen > 0


def test_tables_for_uses_device_and_matches_host():
    from paper_1503_07221_b200 import kernel_weights as K
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=3.95, N=80, p=0)
    dev = K.tables_for(grid)
    host = K.tables_for(grid, device=False)
    assert dev is not host
    for key, tbl in host.tables.items():
        if tbl is None:
            assert dev.tables[key] is None
            continue
        ref = tbl.coeffs
        assert np.max(np.abs(dev.tables[key].coeffs - ref)) <= 1e-13 * np.max(np.abs(ref))
