"""Retarded double-layer potential off the boundary, on the GPU.

Mirrors tdbem.potential (/root/reference/pkg/src/tdbem/potential.py):
  FieldGrid            :24-37  (points, times, validate)
  eval_double_layer    :53-104 (one point, one time; q_far / q_near rules)
  eval_total_field     :107-126 (incident + scattered on a FieldGrid)
plus eval_double_layer_batch, the whole (times x points) grid in one call
(csrc/tdb_potential.cu, C ABI tdb_dlp_eval).  Same arguments and semantics;
the coefficients are the solver's time-major vector (L * M values).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .assembly import _mesh_c, as_product_inputs
from .quadrature import triangle_rule

__all__ = ["FieldGrid", "eval_double_layer", "eval_double_layer_batch", "eval_total_field"]


@dataclass(frozen=True)
class FieldGrid:
    """Evaluation points (off the surface) and times."""

    points: np.ndarray
    times: np.ndarray



def _validate(fieldgrid, mesh, min_dist: float = 1e-8) -> None:
    c = mesh.corners
    for pt in np.atleast_2d(fieldgrid.points):
        d = _point_triangle_distance(np.broadcast_to(pt, (mesh.num_triangles, 3)), c[:, 0], c[:, 1], c[:, 2]).min()
        if d < min_dist:
            raise ValueError(f"field point {pt} is within {min_dist} of the surface")


FieldGrid.validate = _validate  # same check as potential.py:30-37


def _segment_distance(p, a, b):
    ab = b - a
    den = np.sum(ab * ab, axis=1)
    t = np.clip(np.sum((p - a) * ab, axis=1) / np.where(den > 0, den, 1.0), 0.0, 1.0) * (den > 0)
    return np.linalg.norm(p - a - t[:, None] * ab, axis=1)


def _point_triangle_distance(p, v0, v1, v2):
    """Exact point-triangle distance (the reference's mesh.py:323-354 formulas)."""
    e0, e1, w = v1 - v0, v2 - v0, p - v0
    n = np.cross(e0, e1)
    nn = np.sum(n * n, axis=1)
    dplane = np.abs(np.sum(w * n, axis=1)) / np.sqrt(np.where(nn > 0, nn, 1.0))
    d00, d01, d11 = np.sum(e0 * e0, axis=1), np.sum(e0 * e1, axis=1), np.sum(e1 * e1, axis=1)
    d20, d21 = np.sum(w * e0, axis=1), np.sum(w * e1, axis=1)
    den = d00 * d11 - d01 * d01
    ds = np.where(den > 0, den, 1.0)
    u, v = (d11 * d20 - d01 * d21) / ds, (d00 * d21 - d01 * d20) / ds
    inside = (u >= 0) & (v >= 0) & (u + v <= 1) & (den > 0) & (nn > 0)
    edge = np.minimum.reduce([_segment_distance(p, v0, v1), _segment_distance(p, v1, v2),
                              _segment_distance(p, v2, v0)])
    return np.where(inside, dplane, edge)


def eval_double_layer_batch(mesh, grid, coeffs, points, times, q_far: int = 4, q_near: int = 12,
                            ctx: _lib.Context | None = None) -> np.ndarray:
    """u(points[x], times[t]) for every pair; shape (len(times), len(points))."""
    mesh, grid = as_product_inputs(mesh, grid)
    ctx = ctx or _lib.default_context()
    pts = _lib.f64(np.atleast_2d(points))
    tms = _lib.f64(np.atleast_1d(times))
    alpha = _lib.f64(coeffs).ravel()
    if alpha.size != grid.L * mesh.num_vertices:
        raise ValueError(f"coeffs must hold L*M = {grid.L * mesh.num_vertices} values, got {alpha.size}")
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ValueError("points must have shape (n, 3)")
    fx, fw = (_lib.f64(a) for a in triangle_rule(q_far))
    nx, nw = (_lib.f64(a) for a in triangle_rule(q_near))
    out = np.empty((len(tms), len(pts)))
    keep: list = []
    _lib.check(_lib.LIB.tdb_dlp_eval(
        ctx.handle, _lib.C.byref(_mesh_c(mesh, keep)), float(grid.T), int(grid.N), int(grid.p), _lib.ptr(alpha),
        len(pts), _lib.ptr(pts), len(tms), _lib.ptr(tms), len(fw), _lib.ptr(fx), _lib.ptr(fw), len(nw),
        _lib.ptr(nx), _lib.ptr(nw), _lib.ptr(out)), "dlp_eval")
    return out


def eval_double_layer(mesh, grid, coeffs, point, t: float, q_far: int = 4, q_near: int = 12) -> float:
    """Double layer potential at one off-boundary point and time (potential.py:53-104)."""
    return float(eval_double_layer_batch(mesh, grid, coeffs, np.asarray(point, dtype=float)[None, :],
                                         [float(t)], q_far, q_near)[0, 0])


def eval_total_field(wave, mesh, grid, coeffs, fieldgrid: FieldGrid, q_far: int = 4, q_near: int = 12) -> np.ndarray:
    """Incident plus scattered field, shape (n_times, n_points) (potential.py:107-126).

    `wave` is any object with the reference IncidentWave's field(points, t) method."""
    pts = np.atleast_2d(fieldgrid.points)
    times = np.atleast_1d(fieldgrid.times)
    u = eval_double_layer_batch(mesh, grid, coeffs, pts, times, q_far, q_near)
    for a, t in enumerate(times):
        u[a] += np.asarray(wave.field(pts, float(t)), dtype=float)
    return u
