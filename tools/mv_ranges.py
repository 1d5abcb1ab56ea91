"""Matvec time per block range, for the ranges the recursive preconditioner uses
(GPU box).  usage: mv_ranges.py [config]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1503_07221_b200.block_system import assemble_system  # noqa: E402
from paper_1503_07221_b200.configs import get_config  # noqa: E402

cfg = get_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
mesh, grid = cfg.mesh(), cfg.grid()
A = assemble_system(mesh, grid, device=0)
N, M = grid.N, mesh.num_vertices
h = (N + 1) // 2
q = (h + 1) // 2
ranges = [((1, h), (1, h)), ((h + 1, N), (1, h)), ((1, q), (1, q)), ((q + 1, h), (1, q)), ((q + 1, h), (q + 1, h)),
          ((h + 1, h + q), (h + 1, h + q)), ((h + q + 1, N), (h + 1, h + q))]
for rows, cols in ranges:
    x = torch.randn((cols[1] - cols[0] + 1) * M, dtype=torch.float64, device="cuda")
    for _ in range(3):
        A.matvec(x, rows=rows, cols=cols)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        A.matvec(x, rows=rows, cols=cols)
    e1.record()
    e1.synchronize()
    pl = A.matvec_plan(rows, cols)
    print(f"rows{rows} cols{cols}: {e0.elapsed_time(e1) / 20:.4f} ms tiled {pl.tiled_terms} csr {pl.csr_terms}", flush=True)
