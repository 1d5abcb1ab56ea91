"""Solver timings, device vs the reference package (GPU box).

    python tools/solve_compare.py [--out profiles/r02/solve_compare_r02.json]

Device (this repo): FGMRES(50, 2(2,10)) and DGMRES(50, 4, 20) at eps 1e-5 with the
Gaussian-pulse right-hand side, configs 1 and 2 (config 4: FGMRES only) (setup = matvec plans + graph capture,
reported apart).  Reference (tdbem from oracle/_ref/pkg, single process as the
reference runs its solvers): the same solves on its own config-1
system; at config 2 the reference's FGMRES is timed for its first 3 outer steps only
(~10 s per outer step on the host; a full solve is ~180 steps) and reported per step.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def device(c, with_dgmres=True):
    import torch

    from paper_1503_07221_b200 import solvers as S
    from paper_1503_07221_b200.assembly import assemble_rhs, gaussian_pulse_neumann
    from paper_1503_07221_b200.block_system import assemble_system
    from paper_1503_07221_b200.configs import get_config

    cfg = get_config(c)
    mesh, grid = cfg.mesh(), cfg.grid()
    A = assemble_system(mesh, grid)
    b = torch.as_tensor(assemble_rhs(mesh, grid, gaussian_pulse_neumann(mesh))).cuda()
    out = {}
    fc = S.SolverConfig(restart=50, tol=1e-5, max_iter=20000, recursion_depth=2, inner_iterations=(2, 10))
    t0 = time.perf_counter()
    prec = S.recursive_preconditioner(A, fc)
    for _ in range(3):
        prec(b)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    x, h = S.fgmres(lambda v: A.matvec(v), b, fc, precond=prec)
    torch.cuda.synchronize()
    out["fgmres_rec"] = {"seconds": time.perf_counter() - t0, "setup_seconds": setup, "iterations": len(h)}
    if not with_dgmres:
        return out
    dc = S.SolverConfig(restart=50, tol=1e-5, max_iter=40000, deflate_per_restart=4, max_deflation=20)
    A.matvec(b)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, h, st = S.dgmres(lambda v: A.matvec(v), b, dc)
    torch.cuda.synchronize()
    out["dgmres"] = {"seconds": time.perf_counter() - t0, "iterations": len(h), "rank": st.rank}
    return out


def reference(c, fgmres_steps=None):
    from oracle import reference_arm as RA

    RA.import_reference()
    import numpy as np
    from tdbem.assembly import assemble_rhs
    from tdbem.block_system import assemble_system
    from tdbem.solvers import SolverConfig, dgmres, fgmres, recursive_preconditioner

    name, mesh, grid = RA.config_inputs(c)
    mesh.tri_distance_bounds
    mesh.dof_distance_bounds
    A = assemble_system(mesh, grid, workers=os.cpu_count() or 1)
    zmin = float(mesh.vertices[:, 2].min())
    nz = mesh.normals[:, 2]

    def g(X, t, sigma=0.2, t0=1.0):
        nq = len(X) // mesh.num_triangles
        s = t - t0 - (X[:, 2] - zmin)
        return np.repeat(nz, nq) * (-s / sigma**2) * np.exp(-s * s / (2 * sigma * sigma))

    b = assemble_rhs(mesh, grid, g)
    out = {}
    fc = SolverConfig(restart=50, tol=1e-5, max_iter=fgmres_steps or 20000, recursion_depth=2,
                      inner_iterations=(2, 10))
    t0 = time.perf_counter()
    x, h = fgmres(lambda v: A @ v, b, fc, precond=recursive_preconditioner(A, fc))
    dt = time.perf_counter() - t0
    out["fgmres_rec"] = {"seconds": dt, "iterations": len(h), "seconds_per_step": dt / len(h),
                         "complete": fgmres_steps is None}
    if fgmres_steps is None:
        dc = SolverConfig(restart=50, tol=1e-5, max_iter=40000, deflate_per_restart=4, max_deflation=20)
        t0 = time.perf_counter()
        x, h, st = dgmres(lambda v: A @ v, b, dc)
        out["dgmres"] = {"seconds": time.perf_counter() - t0, "iterations": len(h), "rank": st.rank}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "solve_compare_r02.json"))
    args = ap.parse_args()
    res = {"device": {}, "reference": {}}
    for c in (1, 2, 4):
        res["device"][c] = device(c, with_dgmres=c <= 2)
        print("device", c, res["device"][c], flush=True)
    res["reference"][1] = reference(1)
    print("reference 1", res["reference"][1], flush=True)
    res["reference"][2] = reference(2, fgmres_steps=3)
    print("reference 2", res["reference"][2], flush=True)
    res["host_cores"] = os.cpu_count()
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
