"""Scattered-field evaluation on the paper's 257 x 257 = 66049-point grid.

    python tools/field_probe.py [config=2] [times=3]

Plane z = 0 through the sphere's centre, [-2, 2]^2 (points on/near the surface are
skipped as the reference's FieldGrid.validate would reject them), density = the
FGMRES solution of the Gaussian-pulse problem.  Prints the GPU time and the
oracle's time per point on a small sample (the reference's eval_double_layer is
the same per-point numpy algorithm)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_07221_b200 import solvers as S  # noqa: E402
from paper_1503_07221_b200.assembly import assemble_rhs, gaussian_pulse_neumann  # noqa: E402
from paper_1503_07221_b200.block_system import assemble_system  # noqa: E402
from paper_1503_07221_b200.configs import get_config  # noqa: E402
from paper_1503_07221_b200.potential import eval_double_layer_batch  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = get_config(c)
mesh, grid = cfg.mesh(), cfg.grid()
A = assemble_system(mesh, grid, device=0)
b = torch.as_tensor(assemble_rhs(mesh, grid, gaussian_pulse_neumann(mesh))).cuda()
scfg = S.SolverConfig(method="fgmres-recursive", restart=50, tol=1e-5, max_iter=2000, recursion_depth=2,
                      inner_iterations=(2, 10))
x, hist = S.fgmres(lambda v: A.matvec(v), b, scfg, precond=S.recursive_preconditioner(A, scfg))
coeffs = x.cpu().numpy()
g = np.linspace(-2.0, 2.0, 257)
X, Y = np.meshgrid(g, g, indexing="ij")
pts = np.stack([X.ravel(), Y.ravel(), np.zeros(X.size)], axis=1)
rad = np.linalg.norm(pts, axis=1)
pts = pts[np.abs(rad - 1.0) > 0.02]
times = np.linspace(1.0, grid.T, nt)
eval_double_layer_batch(mesh, grid, coeffs, pts[:100], times[:1])  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
u = eval_double_layer_batch(mesh, grid, coeffs, pts, times)
t_gpu = time.perf_counter() - t0
from oracle.potential import eval_double_layer as oracle_dl  # noqa: E402

sample = pts[:: max(1, len(pts) // 20)][:20]
t0 = time.perf_counter()
ref = np.array([oracle_dl(mesh, grid, coeffs, p, float(times[-1])) for p in sample])
t_cpu_pt = (time.perf_counter() - t0) / len(sample)
ug = eval_double_layer_batch(mesh, grid, coeffs, sample, times[-1:])[0]
print(json.dumps({"config": cfg.name, "points": len(pts), "times": nt, "gpu_seconds": round(t_gpu, 3),
                  "gpu_point_times_per_s": len(pts) * nt / t_gpu,
                  "oracle_seconds_per_point_time": round(t_cpu_pt, 4),
                  "oracle_extrapolated_seconds": round(t_cpu_pt * len(pts) * nt, 1),
                  "max_rel_diff_sample": float(np.max(np.abs(ug - ref)) / np.max(np.abs(ref))),
                  "u_range": [float(u.min()), float(u.max())]}))
