"""Time the FGMRES(50, 2(2,10)) recursive solve on config <c> with <iters> outer steps (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1503_07221_b200 import configs, solvers as S
from paper_1503_07221_b200.assembly import assemble_rhs, gaussian_pulse_neumann
from paper_1503_07221_b200.block_system import assemble_system

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
cf = configs.get_config(c)
mesh, grid = cf.mesh(), cf.grid()
A = assemble_system(mesh, grid, device=0)
b = torch.as_tensor(assemble_rhs(mesh, grid, gaussian_pulse_neumann(mesh))).cuda()
cfg = S.SolverConfig(method="fgmres-recursive", restart=50, tol=1e-5, max_iter=iters, recursion_depth=2,
                     inner_iterations=(2, 10))
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, hist = S.fgmres(lambda v: A.matvec(v), b, cfg, precond=S.recursive_preconditioner(A, cfg))
    torch.cuda.synchronize()
    print(f"solve cfg{c}: {time.perf_counter() - t0:.3f} s, {len(hist)} outer steps, rel res {hist[-1]:.3e}")
