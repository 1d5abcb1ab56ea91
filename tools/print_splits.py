"""Print the (R, D, K) evaluation split each table family runs with at configs 1-4 (GPU box)."""
import json
import sys

sys.path.insert(0, ".")
from paper_1503_07221_b200.assembly import DeviceAssembly, build_plan  # noqa: E402
from paper_1503_07221_b200.block_system import canonical_positions  # noqa: E402
from paper_1503_07221_b200.configs import get_config  # noqa: E402
from paper_1503_07221_b200.kernel_weights import tables_for  # noqa: E402

out = {}
for c in (1, 2, 3, 4):
    cfg = get_config(c)
    mesh, grid = cfg.mesh(), cfg.grid()
    plan = build_plan(mesh, grid, tables_for(grid), canonical_positions(grid, mesh.diameter))
    dev = DeviceAssembly(mesh, plan, create_only=True)
    out[c] = {"|".join(k): v for k, v in dev.family_splits().items()}
    del dev
print(json.dumps(out))
