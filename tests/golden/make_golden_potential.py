"""Double-layer potential goldens from the REFERENCE eval_double_layer (build container only).

    python tests/golden/make_golden_potential.py [--refpkg /tmp/refpkg]

potential.npz: the reference's tdbem.potential.eval_double_layer (potential.py:53-104)
on seeded inputs: icosphere(1) (80 triangles), p = 0 (N = 8, T = 2.8) and p = 1
(N = 6, T = 2.5), seeded density coefficients, off-surface points inside and outside
the sphere (some near the surface so the q_near rule is used) and several times.
"""
import argparse
import os
import sys

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--refpkg", default="/tmp/refpkg")
    args = ap.parse_args()
    sys.path.insert(0, os.path.join(args.refpkg, "src"))
    from tdbem.mesh import icosahedron, refine
    from tdbem.potential import eval_double_layer
    from tdbem.temporal_basis import TimeGrid

    mesh = refine(icosahedron(), True)
    rng = np.random.default_rng(11)
    pts = np.concatenate([
        rng.uniform(-0.5, 0.5, (4, 3)),                      # inside
        rng.standard_normal((4, 3)) * 0.4 + [1.6, 0.0, 0.0],  # outside, far
        np.array([[0.0, 0.0, 1.08], [0.0, 0.93, 0.0], [0.7, 0.7, 0.05], [-1.2, 0.3, 0.4]]),  # near
    ])
    out = {"vertices": mesh.vertices, "triangles": mesh.triangles, "points": pts}
    for tag, (T, N, p) in {"p0": (2.8, 8, 0), "p1": (2.5, 6, 1)}.items():
        grid = TimeGrid(T=T, N=N, p=p)
        coeffs = rng.standard_normal(grid.L * mesh.num_vertices)
        times = np.array([0.35, 1.0, 1.7, T - 0.05, T + 0.6])
        vals = np.array([[eval_double_layer(mesh, grid, coeffs, x, float(t)) for x in pts] for t in times])
        out[f"{tag}_grid"] = np.array([T, N, p])
        out[f"{tag}_coeffs"] = coeffs
        out[f"{tag}_times"] = times
        out[f"{tag}_u"] = vals
        # non-default rules
        out[f"{tag}_u_q38"] = np.array([eval_double_layer(mesh, grid, coeffs, x, 1.3, 3, 8) for x in pts])
    np.savez_compressed(os.path.join(OUT, "potential.npz"), **out)
    print({k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
