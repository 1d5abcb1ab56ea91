"""Matvec probe (and ncu target): assemble one config on cuda:0, time full and
preconditioner-shaped partial matvecs.  usage: mv_probe.py [config] [warm]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1503_07221_b200.block_system import assemble_system  # noqa: E402
from paper_1503_07221_b200.configs import get_config  # noqa: E402

cfg = get_config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
mesh, grid = cfg.mesh(), cfg.grid()
A = assemble_system(mesh, grid, device=0)
N, M, np1 = grid.N, mesh.num_vertices, grid.p + 1
h = (N + 1) // 2
q = (h + 1) // 2
ranges = [((1, N), (1, N)), ((h + 1, N), (h + 1, N)), ((h + 1, N), (1, h)), ((1, q), (1, q))]
for rows, cols in ranges:
    x = torch.randn((cols[1] - cols[0] + 1) * np1 * M, dtype=torch.float64, device="cuda")
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
        y = A.matvec(x, rows=rows, cols=cols)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        y = A.matvec(x, rows=rows, cols=cols)
    e1.record()
    e1.synchronize()
    pl = A.matvec_plan(rows, cols)
    ms = e0.elapsed_time(e1) / 20
    print(f"matvec rows{rows} cols{cols}: {ms:.4f} ms  bytes {pl.bytes:.3e} flops {pl.flops:.3e} "
          f"nterms {pl.nterms} tiled {pl.tiled_terms} csr {pl.csr_terms}  {pl.bytes / ms / 1e6:.0f} GB/s", flush=True)
