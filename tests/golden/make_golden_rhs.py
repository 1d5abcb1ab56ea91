"""RHS golden vectors from the REFERENCE assemble_rhs (build container only).

    python tests/golden/make_golden_rhs.py [--refpkg /tmp/refpkg]

rhs.npz: config-1 Gaussian-pulse load vector (SURVEY 8d RHS) and the reference
test_assembly.py:169-209 smooth datum on the two-triangle mesh (N=5, p=1).
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
    from tdbem.assembly import assemble_rhs
    from tdbem.mesh import SurfaceMesh, icosahedron, refine
    from tdbem.temporal_basis import TimeGrid

    m = refine(refine(icosahedron(), True), True)
    zmin = float(m.vertices[:, 2].min())
    nz = m.normals[:, 2]

    def g(X, t, sigma=0.2, t0=1.0):
        nq = len(X) // m.num_triangles
        s = t - t0 - (X[:, 2] - zmin)
        return np.repeat(nz, nq) * (-s / sigma**2) * np.exp(-s * s / (2 * sigma * sigma))

    b1 = assemble_rhs(m, TimeGrid(T=3.9, N=40, p=0), g)
    verts = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [1.0, 1.0, 0.5]])
    tt = SurfaceMesh(verts, np.array([[0, 1, 2], [1, 3, 2]]))

    def gs(X, t):
        return (X[:, 0] + 2 * X[:, 1] - X[:, 2]) * np.sin(3 * t) * t * t * np.exp(-t)

    b2 = assemble_rhs(tt, TimeGrid(T=3.0, N=5, p=1), gs)
    np.savez_compressed(os.path.join(OUT, "rhs.npz"), cfg1_pulse=b1, two_tri_smooth=b2)


if __name__ == "__main__":
    main()
