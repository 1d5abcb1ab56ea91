"""Calibrate the reference arm's row-sampled estimator against FULL reference assemblies.

    python tools/calibrate_reference.py [--configs 1 2] [--out profiles/r02/ref_calibration.json]

For each config: the reference's own assemble_system(workers = all host cores)
with the mesh's distance bounds pre-warmed (untimed), timed
end to end -> units/s; then the reference arm's RowSampler (oracle/reference_arm.py)
for 3 steps -> units/s.  Only the reference package runs (no product import).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import reference_arm as RA  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "ref_calibration.json"))
    args = ap.parse_args()
    RA.import_reference()
    from tdbem.block_system import assemble_system

    res = []
    for c in args.configs:
        name, mesh, grid = RA.config_inputs(c)
        units, npos = RA.full_units(c)
        t0 = time.perf_counter()
        mesh.tri_distance_bounds
        mesh.dof_distance_bounds
        t_bounds = time.perf_counter() - t0
        workers = os.cpu_count() or 1
        t0 = time.perf_counter()
        A = assemble_system(mesh, grid, workers=workers)
        t_full = time.perf_counter() - t0
        assert len(A.unique_blocks) == npos
        rs = RA.RowSampler(c, int(os.environ.get("REF_ROWS", "0")) or {1: 24, 2: 8, 3: 4, 4: 2, 5: 1}[c])
        su, ss = [], []
        for step in range(4):
            u, s = rs.step(rs.prepare(step))
            if step:
                su.append(u)
                ss.append(s)
        r = {"config": name, "units": units, "positions": npos, "workers": workers,
             "full_assemble_system_s": t_full, "full_units_per_s": units / t_full,
             "prewarm_bounds_s": t_bounds, "sampler_units": su, "sampler_s": ss,
             "sampler_units_per_s": sum(su) / sum(ss),
             "sampler_over_full": (sum(su) / sum(ss)) / (units / t_full)}
        print(json.dumps(r), flush=True)
        res.append(r)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
