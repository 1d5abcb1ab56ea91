"""Formats either side of the path: VTU writer byte-identical to
the reference's, the reference BlockHessenbergMatrix export (CPU, reference blocks
from the goldens), and (GPU) the matrix-statistics dump against the stored nnz."""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, golden


def test_write_vtu_byte_identical_to_reference(tmp_path):
    from paper_1503_07221_b200.io import write_vtu

    g = golden("vtu_inputs.npz")
    write_vtu(str(tmp_path / "q.vtu"), g["pts"], g["vals"], (3, 4))
    write_vtu(str(tmp_path / "v.vtu"), g["pts"][:5], g["vals"][:5])
    for mine, ref in (("q.vtu", "field_quad_ref.vtu"), ("v.vtu", "field_vertex_ref.vtu")):
        assert (tmp_path / mine).read_bytes() == open(os.path.join(GOLDEN, ref), "rb").read()


def test_save_coefficients_roundtrip(tmp_path):
    from paper_1503_07221_b200.io import save_coefficients

    x = np.random.default_rng(1).standard_normal(17)
    save_coefficients(str(tmp_path / "coefficients.npy"), x)
    assert np.array_equal(np.load(tmp_path / "coefficients.npy"), x)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference package not present")
def test_reference_matrix_export_matvec():
    import types

    import scipy.sparse as sp

    sys.path.insert(0, "/root/reference/pkg/src")
    import tdbem.block_system  # noqa: F401
    import tdbem.temporal_basis  # noqa: F401

    from paper_1503_07221_b200.io import to_reference_matrix
    from paper_1503_07221_b200.mesh import icosahedron
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    g = golden("blocks_ico_N5_p1.npz")
    grid = TimeGrid(T=2.0, N=5, p=1)
    positions = [tuple(int(v) for v in r) for r in g["positions"]]
    blocks = {}
    for kt, it in positions:
        blocks[(kt, it)] = [[sp.csr_matrix(g[f"b_{kt}_{it}_{m2}_{m1}"]) if f"b_{kt}_{it}_{m2}_{m1}" in g.files
                             else None for m1 in range(2)] for m2 in range(2)]
    mesh = icosahedron()
    A = types.SimpleNamespace(grid=grid, M=mesh.num_vertices, diameter=mesh.diameter, unique_blocks=blocks)
    R = to_reference_matrix(A, tdbem=sys.modules["tdbem"])
    assert type(R).__module__ == "tdbem.block_system"
    assert np.linalg.norm(R.matvec(g["x7"]) - g["y7"]) <= 1e-12 * np.linalg.norm(g["y7"])


@pytest.mark.gpu
def test_matrix_statistics_counts(tmp_path):
    from paper_1503_07221_b200.block_system import assemble_system, plan_distribution
    from paper_1503_07221_b200.io import matrix_statistics, write_matrix_statistics_csv
    from paper_1503_07221_b200.mesh import icosphere
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    mesh, grid = icosphere(2), TimeGrid(T=3.9, N=40, p=0)
    A = assemble_system(mesh, grid)
    plan = plan_distribution(grid, mesh, 4)
    rows = matrix_statistics(A, plan)
    n = write_matrix_statistics_csv(A, str(tmp_path / "stats.csv"), plan)
    assert n == len(rows) and n > 0
    canon = {(r[2], r[3]): r[4] for r in rows}
    assert sum(canon.values()) == A.stats()["nnz_total"]
    assert set(canon) == set(A.unique_blocks)
    assert all(0 <= r[5] < 4 for r in rows)
    from paper_1503_07221_b200.block_system import canonical_position

    logical = sum(1 for kt in range(1, 41) for it in range(1, 41)
                  if not A.is_zero_position(kt, it) and canonical_position(grid, kt, it) in A.unique_blocks)
    assert logical == n
