"""Quarter-range matvec only (the recursive preconditioner's dominant operation); ncu target."""
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
for rows in [(1, q), (q + 1, h), (1, h)]:
    cols = rows
    x = torch.randn((cols[1] - cols[0] + 1) * np1 * M, dtype=torch.float64, device="cuda")
    for _ in range(3):
        y = A.matvec(x, rows=rows, cols=cols)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        y = A.matvec(x, rows=rows, cols=cols)
    e1.record()
    e1.synchronize()
    pl = A.matvec_plan(rows, cols)
    print(f"matvec rows{rows}: {e0.elapsed_time(e1) / 50 * 1000:.1f} us  nterms {pl.nterms} flops {pl.flops:.3e}", flush=True)
