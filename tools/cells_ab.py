"""A/B of the quadrature kernels: default (k_quad_cells for the regular pairs of the
grid families + k_quad for the rest) against TDB_CELLS=0 (k_quad only), same system.

    python tools/cells_ab.py CONFIG [--time]

Each arm runs in its own process (the switch is read at system creation); prints the
largest entry difference relative to each position's max |entry| and the phase times.
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ARM = r'''
import sys, json, numpy as np
sys.path.insert(0, ".")
from paper_1503_07221_b200.configs import get_config
from paper_1503_07221_b200.block_system import assemble_system
cfg = get_config(int(sys.argv[1]))
A = assemble_system(cfg.mesh(), cfg.grid())
dev = A._dev
if len(sys.argv) > 3:
    for _ in range(2):
        dev.rerun()
out = {}
for f in range(len(dev.plan.families)):
    indptr, indices, data = dev.family_arrays(f)
    out[f"p{f}"], out[f"i{f}"], out[f"d{f}"] = indptr, indices, data
np.savez(sys.argv[2], **out)
print("STATS " + json.dumps(dev.stats()))
'''


def run(cfg, cells, path, timed):
    env = dict(os.environ, TDB_CELLS=str(cells))
    cmd = [sys.executable, "-c", ARM, str(cfg), path] + (["t"] if timed else [])
    r = subprocess.run(cmd, env=env, capture_output=True, text=True)
    if r.returncode != 0:
        print(r.stdout[-2000:], r.stderr[-4000:])
        raise SystemExit(1)
    st = [l for l in r.stdout.splitlines() if l.startswith("STATS ")][-1]
    return json.loads(st[6:]), r.stderr


def main():
    cfg = int(sys.argv[1])
    timed = "--time" in sys.argv
    with tempfile.TemporaryDirectory() as td:
        s1, e1 = run(cfg, 1, os.path.join(td, "a.npz"), timed)
        s0, e0 = run(cfg, 0, os.path.join(td, "b.npz"), timed)
        a, b = np.load(os.path.join(td, "a.npz")), np.load(os.path.join(td, "b.npz"))
        worst = 0.0
        nf = len([k for k in a.files if k.startswith("d")])
        for f in range(nf):
            assert np.array_equal(a[f"p{f}"], b[f"p{f}"]) and np.array_equal(a[f"i{f}"], b[f"i{f}"]), f
            da, db = a[f"d{f}"].ravel(), b[f"d{f}"].ravel()
            if da.size == 0:
                continue
            scale = max(np.abs(db).max(), 1e-300)
            err = np.abs(da - db).max() / scale
            print(f"family {f}: nnz {da.size} max|diff|/max|a| {err:.3e} nan {int(np.isnan(da).sum())}")
            worst = max(worst, err)
        keys = ("ms_plan", "ms_quad", "ms_quad_cells", "n_in_cells", "pairs_cells", "ms_finalize", "ms_pattern", "ms_total", "n_in", "units")
        print("cells  ", {k: s1[k] for k in keys})
        print("k_quad ", {k: s0[k] for k in keys})
        print("worst", worst)
        if os.environ.get("TDB_VERBOSE"):
            print(e1[-3000:])


if __name__ == "__main__":
    main()
