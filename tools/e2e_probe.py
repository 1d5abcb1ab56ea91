"""Host-side breakdown of the end-to-end assembly call (GPU box)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1503_07221_b200 import _lib  # noqa: E402
from paper_1503_07221_b200.assembly import DeviceAssembly, build_plan  # noqa: E402
from paper_1503_07221_b200.block_system import assemble_system, canonical_positions, plan_distribution  # noqa: E402
from paper_1503_07221_b200.configs import get_config  # noqa: E402
from paper_1503_07221_b200.kernel_weights import tables_for  # noqa: E402

cfg = get_config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
mesh, grid = cfg.mesh(), cfg.grid()
tables = tables_for(grid)
for rep in range(3):
    T = {}
    t = time.perf_counter()
    pd = plan_distribution(grid, mesh, 1); T["plan_distribution"] = time.perf_counter() - t; t = time.perf_counter()
    pos = canonical_positions(grid, mesh.diameter); T["canonical_positions"] = time.perf_counter() - t; t = time.perf_counter()
    plan = build_plan(mesh, grid, tables, pos); T["build_plan"] = time.perf_counter() - t; t = time.perf_counter()
    ctx = _lib.default_context(0); T["ctx"] = time.perf_counter() - t; t = time.perf_counter()
    dev = DeviceAssembly(mesh, plan, ctx); torch.cuda.synchronize(); T["create+run"] = time.perf_counter() - t; t = time.perf_counter()
    host = [dev.family_arrays(f) for f in range(dev.num_families)]; T["copy_out"] = time.perf_counter() - t; t = time.perf_counter()
    st = dev.stats()
    del dev; torch.cuda.synchronize(); T["destroy"] = time.perf_counter() - t
    print({k: round(v * 1e3, 2) for k, v in T.items()}, "device ms_total", round(st["ms_total"], 2), flush=True)
t = time.perf_counter()
A = assemble_system(mesh, grid, tables=tables, device=0)
host = [A._dev.family_arrays(f) for f in range(A._dev.num_families)]
print("assemble_system+copy ms", round((time.perf_counter() - t) * 1e3, 2))
