"""ORACLE (test infrastructure only): numpy restatement of the reference's
retarded double-layer potential (tdbem.potential.eval_double_layer,
/root/reference/pkg/src/tdbem/potential.py:53-104).

    u(x, t) = -(1/4pi) sum_e sum_q w_q 2|e| (n_e.(x - y_q)/r) (phi(y_q, t - r)/r^2 + phi_t(y_q, t - r)/r)

with r = |x - y_q| and the discrete density phi(y, s) = sum_i b_i(s) sum_a
shape_a(y) alpha[i][tri_e[a]] over the basis functions whose support interval
(open, potential.py:86-88) contains s.  Triangles closer than twice their
longest edge to x use the q_near x q_near collapsed rule, the others q_far x
q_far (potential.py:67-76).  Pinned against tests/golden/potential.npz, which
the reference itself produced (tests/golden/make_golden_potential.py).
"""

from __future__ import annotations

import numpy as np

from paper_1503_07221_b200.quadrature import shape_values, triangle_rule
from paper_1503_07221_b200.temporal_basis import basis_b, decode_flat, support_interval

from .assembly import point_triangle_distance

_INV4PI = 1.0 / (4.0 * np.pi)


def eval_double_layer(mesh, grid, coeffs, point, t, q_far=4, q_near=12):
    m = mesh.num_vertices
    alpha = np.asarray(coeffs, dtype=float).reshape(grid.L, m)
    point = np.asarray(point, dtype=float)
    c = mesh.corners
    diam = np.linalg.norm(c - c[:, [1, 2, 0]], axis=2).max(axis=1)
    rep = np.broadcast_to(point, (mesh.num_triangles, 3))
    near = point_triangle_distance(rep, c[:, 0], c[:, 1], c[:, 2]) < 2.0 * diam
    total = 0.0
    for q, sel in ((q_far, ~near), (q_near, near)):
        if not np.any(sel):
            continue
        pts, w = triangle_rule(q)
        cs = c[sel]
        X = cs[:, None, 0] + pts[None, :, 0, None] * (cs[:, 1] - cs[:, 0])[:, None] \
            + pts[None, :, 1, None] * (cs[:, 2] - cs[:, 1])[:, None]
        wx = w[None, :] * 2.0 * mesh.areas[sel][:, None]
        sh = shape_values(pts)
        tri = mesh.triangles[sel]
        d = point[None, None, :] - X
        r = np.sqrt(np.sum(d * d, axis=2))
        ndotd = np.sum(mesh.normals[sel][:, None, :] * d, axis=2)
        tret = t - r
        phi = np.zeros_like(r)
        phit = np.zeros_like(r)
        for i in range(1, grid.L + 1):
            lo, hi = support_interval(grid, decode_flat(grid, i).timestep)
            mask = (tret > lo) & (tret < hi)
            if not np.any(mask):
                continue
            dof = sh @ alpha[i - 1][tri].T  # (nq, E_sel)
            dof = dof.T
            phi[mask] += basis_b(grid, i, tret[mask]) * dof[mask]
            phit[mask] += basis_b(grid, i, tret[mask], deriv=1) * dof[mask]
        kern = ndotd / r * (phi / r**2 + phit / r)
        total += -_INV4PI * float(np.sum(wx * kern))
    return total
