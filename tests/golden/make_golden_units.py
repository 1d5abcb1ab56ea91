"""Per-position admissible-unit counts of a BASELINE config from the REFERENCE's primitives.

    python tests/golden/make_golden_units.py --config 5 [--workers 8]

Build container only.  A unit is one admissible (triangle pair, canonical
position): the pair (ex, ey) is admissible at (kt, it) iff
tmin[ex, ey] <= shi and tmax[ex, ey] >= slo with [slo, shi] = psi_support
(ref/assembly.py:167-184, ref/kernel_weights.py:381-385).  The bounds are the
reference's own (ref/mesh.py:357-391, evaluated in row chunks by
refhelpers.pair_bounds, bit-identical to the dense evaluation), the positions
its own enumeration (ref/block_system.py:249-258), the supports its own
psi_support.  Positions with is_zero_pair have no units (ref/assembly.py:175).

Writes units_cfg{c}.npz: positions (P, 2), units (P,).  With --sample-rows K
it writes units_cfg{c}_rows.npz instead: the counts restricted to the test
triangles in the stars of K seeded test vertices (the row block a single GPU
can assemble at config 5), with those vertices.

Config 5 (full): 6 610 143 148 units - the product's count.  SURVEY 8d's
6 609 879 544 was not the reference's block_pattern count (its config-1 figure,
2 193 464, also differs from the reference's 2 194 144, tests/golden/blocks_cfg1.npz).
"""

from __future__ import annotations

import argparse
import os
import time

import numpy as np

import refhelpers as R

OUT = os.path.dirname(os.path.abspath(__file__))
_G = {}


def _init(c):
    R.prepare()
    mesh, grid = R.config_inputs(c)
    _G["mesh"], _G["grid"] = mesh, grid


def _count_chunk(args):
    r0, r1, slo, shi = args
    mesh = _G["mesh"]
    E = mesh.num_triangles
    cols = _G.get("cols")
    if cols is None:  # all ordered pairs, x-triangle rows r0..r1
        ii = np.repeat(np.arange(r0, r1), E)
        jj = np.tile(np.arange(E), r1 - r0)
    else:  # test triangles cols[r0:r1] against every x-triangle
        ii = np.tile(np.arange(E), r1 - r0)
        jj = np.repeat(cols[r0:r1], E)
    tmin, tmax = R.pair_bounds(mesh.corners, mesh.triangles, ii, jj)
    # per position: #(tmin <= shi) - #(tmin <= shi and tmax < slo); use sorted keys
    out = np.zeros(len(slo), dtype=np.int64)
    order = np.argsort(tmin, kind="stable")
    tmin_s = tmin[order]
    tmax_s = tmax[order]
    for k in range(len(slo)):
        n = np.searchsorted(tmin_s, shi[k], side="right")
        out[k] = n - np.count_nonzero(tmax_s[:n] < slo[k])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--rows", type=int, default=64)
    ap.add_argument("--sample-rows", type=int, default=0)
    args = ap.parse_args()
    R.prepare()
    from tdbem.kernel_weights import is_zero_pair, psi_support

    mesh, grid = R.config_inputs(args.config)
    positions = R.canonical_positions(mesh, grid)
    live = [p for p in positions if not is_zero_pair(grid, *p)]
    sup = np.array([psi_support(grid, kt, it) for kt, it in live], dtype=np.float64).reshape(-1, 2)
    slo, shi = sup[:, 0].copy(), sup[:, 1].copy()
    E = mesh.num_triangles
    extra = {}
    if args.sample_rows:
        rng = np.random.default_rng(2000 + args.config)
        vrows = np.sort(rng.choice(mesh.num_vertices, args.sample_rows, replace=False))
        cols = np.flatnonzero(np.isin(mesh.triangles, vrows).any(axis=1))
        _G["cols"] = cols
        extra = dict(rows=vrows, test_triangles=cols)
        chunks = [(r0, min(len(cols), r0 + 8), slo, shi) for r0 in range(0, len(cols), 8)]
    else:
        chunks = [(r0, min(E, r0 + args.rows), slo, shi) for r0 in range(0, E, args.rows)]
    t0 = time.time()
    import multiprocessing as mp

    total = np.zeros(len(live), dtype=np.int64)
    init = (lambda c: (_init(c), _G.update(cols=extra.get("test_triangles")))) if extra else _init
    with mp.get_context("fork").Pool(args.workers, initializer=init, initargs=(args.config,)) as pool:
        for i, part in enumerate(pool.imap_unordered(_count_chunk, chunks)):
            total += part
            if i % 20 == 0:
                print(f"{i + 1}/{len(chunks)} chunks, {time.time() - t0:.0f} s", flush=True)
    units = np.zeros(len(positions), dtype=np.int64)
    idx = {p: k for k, p in enumerate(positions)}
    for k, p in enumerate(live):
        units[idx[p]] = total[k]
    name = f"units_cfg{args.config}" + ("_rows" if args.sample_rows else "") + ".npz"
    np.savez_compressed(os.path.join(OUT, name), positions=np.array(positions),
                        units=units, mesh_digest=R.mesh_digest(mesh.vertices, mesh.triangles),
                        diameter=np.array([mesh.diameter]), **extra)
    print("config", args.config, "positions", len(positions), "units", int(units.sum()),
          f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
