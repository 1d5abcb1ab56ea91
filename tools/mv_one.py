"""Time one matvec range repeatedly (ncu target).  usage: mv_one.py config rlo rhi clo chi [reps]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1503_07221_b200.block_system import assemble_system  # noqa: E402
from paper_1503_07221_b200.configs import get_config  # noqa: E402

c, rlo, rhi, clo, chi = (int(v) for v in sys.argv[1:6])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 20
cfg = get_config(c)
mesh, grid = cfg.mesh(), cfg.grid()
A = assemble_system(mesh, grid, device=0)
x = torch.randn((chi - clo + 1) * (grid.p + 1) * mesh.num_vertices, dtype=torch.float64, device="cuda")
for _ in range(3):
    A.matvec(x, rows=(rlo, rhi), cols=(clo, chi))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    A.matvec(x, rows=(rlo, rhi), cols=(clo, chi))
e1.record()
e1.synchronize()
pl = A.matvec_plan((rlo, rhi), (clo, chi))
print(f"rows({rlo},{rhi}) cols({clo},{chi}): {e0.elapsed_time(e1) / reps:.4f} ms tiled {pl.tiled_terms} "
      f"csr {pl.csr_terms} bytes {pl.bytes:.3e} flops {pl.flops:.3e}", flush=True)
