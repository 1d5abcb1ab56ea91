"""Block fill factors of the inner-family lag blocks (matvec storage design probe, GPU box).
usage: fill_probe.py config"""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1503_07221_b200.assembly import DeviceAssembly, build_plan  # noqa: E402
from paper_1503_07221_b200.block_system import canonical_positions  # noqa: E402
from paper_1503_07221_b200.configs import get_config  # noqa: E402
from paper_1503_07221_b200.kernel_weights import tables_for  # noqa: E402

cfg = get_config(int(sys.argv[1]))
mesh, grid = cfg.mesh(), cfg.grid()
plan = build_plan(mesh, grid, tables_for(grid), canonical_positions(grid, mesh.diameter))
D = DeviceAssembly(mesh, plan)
M = mesh.num_vertices
V = mesh.vertices
# Morton order of the vertices
q = np.clip(((V - V.min(0)) / (V.max(0) - V.min(0) + 1e-12) * 1023).astype(np.int64), 0, 1023)
def spread(x):
    out = np.zeros_like(x)
    for b in range(10):
        out |= ((x >> b) & 1) << (3 * b)
    return out
code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
perm = np.argsort(code, kind="stable")  # new index -> old vertex
inv = np.empty(M, np.int64); inv[perm] = np.arange(M)
fi = [i for i, f in enumerate(plan.families) if f.kinds == ("inner", "inner")][0]
indptr, indices, data = D.family_arrays(fi)
npos = len(plan.families[fi].positions)
tot = dict()
for s in range(npos):
    rows = np.repeat(np.arange(M), np.diff(indptr[s * M:(s + 1) * M + 1]))
    cols = indices[indptr[s * M]:indptr[(s + 1) * M]].astype(np.int64)
    for name, (r, c) in {"natural": (rows, cols), "morton": (inv[rows], inv[cols])}.items():
        for R, C in [(4, 1), (8, 1), (8, 4), (4, 4)]:
            key = (name, R, C)
            blocks = np.unique((r // R) * (M + 1) + c // C)
            t = tot.setdefault(key, [0, 0])
            t[0] += len(rows)
            t[1] += len(blocks) * R * C
for key, (nnz, slots) in sorted(tot.items()):
    print(f"{key}: fill {nnz / slots:.3f}  (nnz {nnz}, block slots {slots})")
print("nnz per row per lag", tot[("natural", 4, 1)][0] / (npos * M))
