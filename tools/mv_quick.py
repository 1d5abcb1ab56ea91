"""Quarter / half / full matvec times at a config: python tools/mv_quick.py [CONFIG]"""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1503_07221_b200.configs import get_config
from paper_1503_07221_b200.block_system import assemble_system
cfg = get_config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
A = assemble_system(cfg.mesh(), cfg.grid()); N = cfg.N; M = A.M
x = torch.randn(N * M, dtype=torch.float64, device="cuda")
q = ((N + 1) // 2 + 1) // 2; h = (N + 1) // 2
for name, rows, cols in (("quarter", (1, q), (1, q)), ("half", (1, h), (1, h)), ("offdiag", (h + 1, N), (1, h)), ("full", (1, N), (1, N))):
    xs = x[: (cols[1] - cols[0] + 1) * M].contiguous()
    for _ in range(5): A.matvec(xs, rows=rows, cols=cols)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(50): A.matvec(xs, rows=rows, cols=cols)
    torch.cuda.synchronize(); print(name, rows, cols, f"{(time.perf_counter() - t0) / 50 * 1e3:.4f} ms")
