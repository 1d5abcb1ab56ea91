"""Solver golden vectors from the REFERENCE package (build container only).

    python tests/golden/make_golden_solvers.py [--refpkg /tmp/refpkg]

Writes solvers.npz: reference gmres / dgmres / fgmres + recursive preconditioner
solutions and iteration counts on the two-triangle system of the reference's
tests/test_solvers.py:152-189 (N=6, p=1), plus its random well-conditioned
system (tests/test_solvers.py:22-26).
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
    from tdbem.block_system import assemble_system
    from tdbem.mesh import SurfaceMesh
    from tdbem.solvers import SolverConfig, dgmres, fgmres, gmres, recursive_preconditioner
    from tdbem.temporal_basis import TimeGrid

    out = {}
    verts = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [1.0, 1.0, 0.5]])
    mesh = SurfaceMesh(verts, np.array([[0, 1, 2], [1, 3, 2]]))
    grid = TimeGrid(T=3.0, N=6, p=1)
    A = assemble_system(mesh, grid, workers=1)
    b = np.random.default_rng(9).standard_normal(A.shape[0])
    out["b9"] = b
    cfg = SolverConfig(restart=40, tol=1e-8, max_iter=2000)
    x, h = gmres(lambda v: A @ v, b, cfg)
    out["gmres_x"], out["gmres_hist"] = x, np.array(h)
    cfg = SolverConfig(restart=40, tol=1e-8, max_iter=2000, recursion_depth=2, inner_iterations=(2, 6))
    x, h = fgmres(lambda v: A @ v, b, cfg, precond=recursive_preconditioner(A, cfg))
    out["frec_x"], out["frec_hist"] = x, np.array(h)
    cfg = SolverConfig(restart=40, tol=1e-12, max_iter=4000, recursion_depth=2, inner_iterations=(2, 6))
    x, h = fgmres(lambda v: A @ v, b, cfg, precond=recursive_preconditioner(A, cfg))
    out["frec12_x"], out["frec12_hist"] = x, np.array(h)
    cfg = SolverConfig(restart=20, tol=1e-12, max_iter=4000, deflate_per_restart=2, max_deflation=8)
    x, h, st = dgmres(lambda v: A @ v, b, cfg)
    out["dgm_x"], out["dgm_hist"], out["dgm_rank"] = x, np.array(h), np.array([st.rank])
    # random well-conditioned system
    rng = np.random.default_rng(0)
    n = 200
    M = np.eye(n) + (0.5 / np.sqrt(n)) * rng.standard_normal((n, n))
    bb = rng.standard_normal(n)
    out["rand_A"], out["rand_b"] = M, bb
    x, h = gmres(lambda v: M @ v, bb, SolverConfig(restart=50, tol=1e-12))
    out["rand_gmres_x"], out["rand_gmres_hist"] = x, np.array(h)
    x, h, st = dgmres(lambda v: M @ v, bb, SolverConfig(restart=20, tol=1e-12, deflate_per_restart=2,
                                                       max_deflation=8))
    out["rand_dgm_x"], out["rand_dgm_hist"] = x, np.array(h)
    np.savez_compressed(os.path.join(OUT, "solvers.npz"), **out)


if __name__ == "__main__":
    main()
