"""One rank's share of a row-block-sharded assembly, run on one GPU.

    python tools/rank_share.py [config=5] [world=8] [rank=0]

Only one GPU is available to this build, so the 8-GPU configuration-5 stress
test is measured rank by rank: rank r's owned test-vertex rows (distributed.
partition_rows) are assembled on cuda:0 exactly as bench.py --gpus 8 would on
GPU r (no communication in assembly), and a full-range local matvec is timed
with an emulated all-gathered iterate.  Prints one JSON line.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_07221_b200 import _lib  # noqa: E402
from paper_1503_07221_b200.assembly import DeviceAssembly, build_plan  # noqa: E402
from paper_1503_07221_b200.block_system import canonical_positions  # noqa: E402
from paper_1503_07221_b200.configs import get_config  # noqa: E402
from paper_1503_07221_b200.distributed import DistributedBlockHessenbergMatrix, partition_rows  # noqa: E402
from paper_1503_07221_b200.kernel_weights import tables_for  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 5
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = get_config(c)
t0 = time.perf_counter()
mesh, grid = cfg.mesh(), cfg.grid()
tables = tables_for(grid)
plan = build_plan(mesh, grid, tables, canonical_positions(grid, mesh.diameter))
rows, tests = partition_rows(mesh, world)
t_host = time.perf_counter() - t0
ctx = _lib.default_context(0)
free0, total = torch.cuda.mem_get_info()
t0 = time.perf_counter()
D = DeviceAssembly(mesh, plan, ctx, rows=rows[rank], create_only=True)
torch.cuda.synchronize()
t_create = time.perf_counter() - t0
runs = []
for _ in range(3):
    D.rerun()
    runs.append(D.stats())
free1, _ = torch.cuda.mem_get_info()
st = runs[-1]
out = {
    "config": cfg.name, "world": world, "rank": rank, "rows": int(len(rows[rank])),
    "test_triangles": int(len(tests[rank])), "E": mesh.num_triangles, "M": mesh.num_vertices, "N": grid.N,
    "units_rank": int(sum(st["units_case"])), "units_primary": int(st["units_primary"]),
    "n_in": int(st["n_in"]), "ms_total": [round(r["ms_total"], 2) for r in runs],
    "phases_ms": {k: round(v, 2) for k, v in st.items() if k.startswith("ms_")},
    "units_per_s": sum(st["units_case"]) / (st["ms_total"] * 1e-3),
    "device_bytes_in_use_GB": round((free0 - free1) / 1e9, 2), "hbm_total_GB": round(total / 1e9, 1),
    "host_setup_s": round(t_host, 2), "create_s": round(t_create, 2),
}
del D
torch.cuda.empty_cache()
# local full-range matvec of this rank with an emulated all-gathered iterate
A = DistributedBlockHessenbergMatrix(mesh, grid, rows, rank, ctx=ctx, tables=tables,
                                     gather=lambda t: t.unsqueeze(0).expand(world, *t.shape).contiguous())
xl = torch.randn(grid.L * A.M, dtype=torch.float64, device="cuda")
for _ in range(2):
    y = A.matvec(xl)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    y = A.matvec(xl)
e1.record()
e1.synchronize()
out["matvec_ms_local_incl_emulated_gather"] = round(e0.elapsed_time(e1) / 5, 3)
print(json.dumps(out))
