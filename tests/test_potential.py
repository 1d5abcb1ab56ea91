"""Retarded double-layer potential (reference potential.py:53-126).

CPU: the numpy oracle (oracle/potential.py) against the reference's own values
(tests/golden/potential.npz, tests/golden/make_golden_potential.py).
GPU: the device path (csrc/tdb_potential.cu through the C ABI) against the same
goldens and against the oracle on a larger seeded case (config-1 mesh, p = 0).
Tolerance: 1e-12 of the largest |u| of the case (the kernel sums in another order).
"""

import numpy as np
import pytest

from conftest import golden


def _mesh_grid(g, tag):
    from paper_1503_07221_b200.mesh import SurfaceMesh
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    T, N, p = g[f"{tag}_grid"]
    return SurfaceMesh(g["vertices"], g["triangles"]), TimeGrid(T=float(T), N=int(N), p=int(p))


@pytest.mark.parametrize("tag", ["p0", "p1"])
def test_oracle_matches_reference_golden(tag):
    from oracle.potential import eval_double_layer

    g = golden("potential.npz")
    mesh, grid = _mesh_grid(g, tag)
    u = np.array([[eval_double_layer(mesh, grid, g[f"{tag}_coeffs"], x, float(t)) for x in g["points"]]
                  for t in g[f"{tag}_times"]])
    ref = g[f"{tag}_u"]
    assert np.max(np.abs(u - ref)) <= 1e-14 * np.max(np.abs(ref))
    u2 = np.array([eval_double_layer(mesh, grid, g[f"{tag}_coeffs"], x, 1.3, 3, 8) for x in g["points"]])
    assert np.max(np.abs(u2 - g[f"{tag}_u_q38"])) <= 1e-14 * np.max(np.abs(g[f"{tag}_u_q38"]))


def test_field_grid_validation():
    from paper_1503_07221_b200.mesh import icosphere
    from paper_1503_07221_b200.potential import FieldGrid

    m = icosphere(1)
    FieldGrid(np.array([[0.0, 0.0, 0.2], [2.0, 0.0, 0.0]]), np.array([1.0])).validate(m)
    with pytest.raises(ValueError):
        FieldGrid(np.array([m.vertices[3]]), np.array([1.0])).validate(m)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["p0", "p1"])
def test_device_matches_reference_golden(tag):
    from paper_1503_07221_b200.potential import eval_double_layer, eval_double_layer_batch

    g = golden("potential.npz")
    mesh, grid = _mesh_grid(g, tag)
    u = eval_double_layer_batch(mesh, grid, g[f"{tag}_coeffs"], g["points"], g[f"{tag}_times"])
    ref = g[f"{tag}_u"]
    assert np.max(np.abs(u - ref)) <= 1e-12 * np.max(np.abs(ref))
    u2 = np.array([eval_double_layer(mesh, grid, g[f"{tag}_coeffs"], x, 1.3, 3, 8) for x in g["points"]])
    assert np.max(np.abs(u2 - g[f"{tag}_u_q38"])) <= 1e-12 * np.max(np.abs(g[f"{tag}_u_q38"]))


@pytest.mark.gpu
def test_device_matches_oracle_cfg1_and_total_field():
    from oracle.potential import eval_double_layer as oracle_dl
    from paper_1503_07221_b200.mesh import icosphere
    from paper_1503_07221_b200.potential import FieldGrid, eval_double_layer_batch, eval_total_field
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    mesh, grid = icosphere(2), TimeGrid(T=3.9, N=40, p=0)
    rng = np.random.default_rng(5)
    coeffs = rng.standard_normal(grid.L * mesh.num_vertices)
    pts = np.concatenate([rng.uniform(-0.6, 0.6, (3, 3)), rng.standard_normal((3, 3)) * 0.3 + [0, 0, 1.9],
                          np.array([[0.0, 0.0, 1.04], [0.98, 0.0, 0.0]])])
    times = np.array([0.5, 2.0, 3.7])
    u = eval_double_layer_batch(mesh, grid, coeffs, pts, times)
    ref = np.array([[oracle_dl(mesh, grid, coeffs, x, float(t)) for x in pts] for t in times])
    assert np.max(np.abs(u - ref)) <= 1e-12 * np.max(np.abs(ref))

    class Wave:  # any object with field(points, t), like the reference's IncidentWave
        def field(self, p, t):
            return np.sin(t - p[:, 2])

    tot = eval_total_field(Wave(), mesh, grid, coeffs, FieldGrid(pts, times))
    assert np.allclose(tot - u, np.sin(times[:, None] - pts[None, :, 2]), rtol=0, atol=1e-15)
