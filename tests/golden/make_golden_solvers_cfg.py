"""Solver goldens from the REFERENCE package at config 1 and acceptance criterion 7 (build container only).

    python tests/golden/make_golden_solvers_cfg.py

solvers_cfg.npz:
  config 1 (icosphere x2, dt 0.1, N 40, p 0; SURVEY 8d solve-parity protocol), the
  reference's own assembled system and the Gaussian-pulse load vector of rhs.npz:
    frec5_*   FGMRES(50, 2(2,10)), eps 1e-5   (x, history)
    frec12_*  FGMRES(50, 2(2,10)), eps 1e-12
    dgm12_*   DGMRES(50, 4, 20),   eps 1e-12  (x, history, deflation rank)
    dgm5_hist DGMRES(50, 4, 20),   eps 1e-5   (history only: not reproducible)
  acceptance criterion 7 (ref tests/test_acceptance.py:337-360: sphere320.off, T 6,
  N 20, p 1, b = assemble_rhs of sin(3t) t^2 e^-t, eps 1e-5):
    c7_gmres_*, c7_dgmres_*, c7_frec_*  (x, history)
"""
import os
import sys
import time

import numpy as np

import refhelpers as R

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    R.prepare()
    from tdbem.assembly import assemble_rhs
    from tdbem.block_system import assemble_system
    from tdbem.mesh import load_mesh
    from tdbem.solvers import SolverConfig, dgmres, fgmres, gmres, recursive_preconditioner

    out = {}
    t0 = time.time()
    mesh, grid = R.config_inputs(1)
    A = assemble_system(mesh, grid, workers=8)
    b = np.load(os.path.join(OUT, "rhs.npz"))["cfg1_pulse"]
    print(f"cfg1 assembled {time.time() - t0:.0f} s", flush=True)
    for tol, tag in ((1e-5, "frec5"), (1e-12, "frec12")):
        cfg = SolverConfig(restart=50, tol=tol, max_iter=20000, recursion_depth=2, inner_iterations=(2, 10))
        x, h = fgmres(lambda v: A @ v, b, cfg, precond=recursive_preconditioner(A, cfg))
        out[f"{tag}_x"], out[f"{tag}_hist"] = x, np.array(h)
        print(tag, len(h), f"{time.time() - t0:.0f} s", flush=True)
    for tol, tag in ((1e-12, "dgm12"), (1e-5, "dgm5")):
        cfg = SolverConfig(restart=50, tol=tol, max_iter=40000, deflate_per_restart=4, max_deflation=20)
        x, h, st = dgmres(lambda v: A @ v, b, cfg)
        out[f"{tag}_hist"] = np.array(h)
        if tag == "dgm12":
            out["dgm12_x"], out["dgm12_rank"] = x, np.array([st.rank])
        print(tag, len(h), f"{time.time() - t0:.0f} s", flush=True)

    from tdbem.temporal_basis import TimeGrid

    s320 = load_mesh(os.path.join(R.REFPKG, "meshes", "sphere320.off"))
    g7 = TimeGrid(T=6.0, N=20, p=1)
    A7 = assemble_system(s320, g7, workers=8)
    b7 = assemble_rhs(s320, g7, lambda X, t: np.full(len(X), np.sin(3.0 * t) * t * t * np.exp(-t)))
    out["c7_b"] = b7
    print(f"criterion 7 system {time.time() - t0:.0f} s", flush=True)
    x, h = gmres(lambda v: A7 @ v, b7, SolverConfig(restart=50, tol=1e-5, max_iter=20000))
    out["c7_gmres_x"], out["c7_gmres_hist"] = x, np.array(h)
    x, h, _ = dgmres(lambda v: A7 @ v, b7, SolverConfig(restart=50, tol=1e-5, max_iter=20000, deflate_per_restart=4))
    out["c7_dgmres_x"], out["c7_dgmres_hist"] = x, np.array(h)
    cfg = SolverConfig(restart=50, tol=1e-5, max_iter=20000, recursion_depth=2, inner_iterations=(2, 10))
    x, h = fgmres(lambda v: A7 @ v, b7, cfg, precond=recursive_preconditioner(A7, cfg))
    out["c7_frec_x"], out["c7_frec_hist"] = x, np.array(h)
    print("criterion 7 iterations", len(out["c7_gmres_hist"]), len(out["c7_dgmres_hist"]), len(h),
          f"{time.time() - t0:.0f} s", flush=True)
    np.savez_compressed(os.path.join(OUT, "solvers_cfg.npz"), **out)


if __name__ == "__main__":
    main()
