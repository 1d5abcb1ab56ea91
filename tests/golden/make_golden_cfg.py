"""Reference blocks of the BASELINE configs 2-4 (build container only).

    python tests/golden/make_golden_cfg.py --config 2 [--workers 8]

Everything is computed by the REFERENCE package's own assemble_subblocks
(ref/assembly.py:240-306) on the configuration's mesh and grid; only the
distance bounds are pre-populated (the mesh's cached properties, as a
pre-warmed reference run does) with values from the reference's own
primitives (refhelpers.pair_bounds, bit-identical to ref/mesh.py:357-391).

Two kinds of evidence, sized to stay small in git:

* row samples at EVERY canonical position: `nsum` test vertices (seeded), per
  (position, row) the nnz, a hash of the column set, sum |a|, sum a x7 (x7 =
  default_rng(7) normal), and the full CSR entries of the first `nfull` rows.
  The reference is run on a row-restricted copy of the mesh: pairs whose test
  triangle is not in a sampled vertex's star are made inadmissible (so the
  sampled rows are complete and nothing else is computed), plus the touching
  pair of largest tmax per case, which keeps n_rad = its global value
  (ref/assembly.py:281-287, SURVEY finding 6).
* full-block checksums at selected positions of every family (small, middle
  and cutoff lags, the singletons): per row nnz, column hash, sum |a|, sum a x7.

Output: blocks_cfg{c}.npz.
"""

from __future__ import annotations

import argparse
import os
import time

import numpy as np

import refhelpers as R

OUT = os.path.dirname(os.path.abspath(__file__))
_G = {}


def col_hash(cols: np.ndarray) -> np.uint64:
    """Order-independent 64-bit hash of a column set (splitmix64 per id, summed mod 2^64)."""
    z = cols.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        return np.uint64(np.sum(z, dtype=np.uint64))


def row_stats(S, rows, x):
    cnt = np.diff(S.indptr)[rows].astype(np.int32)
    h = np.zeros(len(rows), dtype=np.uint64)
    ab = np.zeros(len(rows))
    ax = np.zeros(len(rows))
    for k, j in enumerate(rows):
        c = S.indices[S.indptr[j]:S.indptr[j + 1]]
        v = S.data[S.indptr[j]:S.indptr[j + 1]]
        h[k] = col_hash(c)
        ab[k] = np.abs(v).sum()
        ax[k] = v @ x[c]
    return cnt, h, ab, ax


def family_key(grid, kt, it):
    kind = lambda t: 0 if t == 1 else (2 if t == grid.N else 1)
    return kind(it), kind(kt)


def select_positions(grid, positions):
    fam = {}
    for kt, it in positions:
        fam.setdefault(family_key(grid, kt, it), []).append((kt, it))
    sel = []
    for key in sorted(fam):
        pos = sorted(fam[key], key=lambda p: p[0] - p[1])
        n = len(pos)
        pick = sorted({0, 1, 2, n // 2, n - 2, n - 1} & set(range(n)))
        sel += [pos[i] for i in pick]
    return sorted(set(sel))


def _job(args):
    which, kt, it = args
    from tdbem.assembly import assemble_subblocks

    mesh = _G["restricted" if which == "rows" else "full"]
    S = assemble_subblocks(mesh, _G["grid"], _G["tabs"], kt, it)[0][0].tocsr()
    S.sort_indices()
    x = _G["x"]
    if which == "rows":
        rows = _G["sum_rows"]
        st = row_stats(S, rows, x)
        fr = _G["full_rows"]
        ent = [(S.indices[S.indptr[j]:S.indptr[j + 1]].astype(np.int32), S.data[S.indptr[j]:S.indptr[j + 1]].copy())
               for j in fr]
        mx = max([np.abs(S.data[S.indptr[j]:S.indptr[j + 1]]).max(initial=0.0) for j in rows])
        return which, (kt, it), st, ent, mx
    st = row_stats(S, np.arange(S.shape[0]), x)
    return which, (kt, it), st, None, (np.abs(S.data).max() if S.nnz else 0.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--nsum", type=int, default=48)
    ap.add_argument("--nfull", type=int, default=3)
    ap.add_argument("--no-full", action="store_true")
    args = ap.parse_args()
    t0 = time.time()
    R.prepare()
    from tdbem.kernel_weights import tables_for
    from tdbem.mesh import SurfaceMesh

    c = args.config
    mesh, grid = R.config_inputs(c)
    E, M = mesh.num_triangles, mesh.num_vertices
    positions = R.canonical_positions(mesh, grid)
    rng = np.random.default_rng(1000 + c)
    sum_rows = np.sort(rng.choice(M, args.nsum, replace=False))
    full_rows = sum_rows[rng.choice(len(sum_rows), args.nfull, replace=False)]
    full_rows.sort()
    tris = mesh.triangles
    in_star = np.isin(tris, sum_rows).any(axis=1)
    S_tri = np.flatnonzero(in_star)
    print(f"config {c}: E={E} M={M} positions={len(positions)} sampled rows={len(sum_rows)} "
          f"test triangles={len(S_tri)}", flush=True)

    # bounds: columns S_tri (admissibility, tmin[ex, ey]) and rows S_tri (dof bounds)
    ii = np.repeat(np.arange(E), len(S_tri))
    jj = np.tile(S_tri, E)
    cmin, cmax = R.pair_bounds(mesh.corners, tris, ii, jj)
    rmin, rmax = R.pair_bounds(mesh.corners, tris, jj, ii)
    # largest-tmax touching pair per case (keeps the reference's n_rad)
    share = {}
    for e in range(E):
        for v in tris[e]:
            share.setdefault(int(v), []).append(e)
    cand = set()
    for v, es in share.items():
        for a in es:
            for b in es:
                cand.add((a, b))
    cand = np.array(sorted(cand))
    tmin_c, tmax_c = R.pair_bounds(mesh.corners, tris, cand[:, 0], cand[:, 1])
    nshared = np.array([len(set(tris[a]) & set(tris[b])) for a, b in cand])
    extra = []
    for ns in (3, 2, 1):
        m = np.flatnonzero(nshared == ns)
        k = m[np.argmax(tmax_c[m])]
        extra.append((int(cand[k, 0]), int(cand[k, 1]), tmin_c[k], tmax_c[k]))

    tmin = np.full((E, E), np.inf)
    tmax = np.full((E, E), -np.inf)
    tmin[ii, jj], tmax[ii, jj] = cmin, cmax
    both_min, both_max = tmin.copy(), tmax.copy()
    both_min[jj, ii], both_max[jj, ii] = rmin, rmax
    for a, b, lo, hi in extra:
        tmin[a, b], tmax[a, b] = lo, hi
        both_min[a, b], both_max[a, b] = lo, hi
    tmp = SurfaceMesh(mesh.vertices, tris)
    tmp.__dict__["tri_distance_bounds"] = (both_min, both_max)
    dofb = type(mesh).dof_distance_bounds.func(tmp)
    restricted = SurfaceMesh(mesh.vertices, tris)
    restricted.__dict__["tri_distance_bounds"] = (tmin, tmax)
    restricted.__dict__["dof_distance_bounds"] = dofb
    del tmp, both_min, both_max
    print(f"restricted bounds ready {time.time() - t0:.0f} s", flush=True)

    sel = [] if args.no_full else select_positions(grid, positions)
    if sel:
        fmin, fmax = R.full_bounds(mesh)
        mesh.__dict__["tri_distance_bounds"] = (fmin, fmax)
        mesh.dof_distance_bounds
        print(f"full bounds ready {time.time() - t0:.0f} s", flush=True)

    _G.update(restricted=restricted, full=mesh, grid=grid, tabs=tables_for(grid),
              x=np.random.default_rng(7).standard_normal(M), sum_rows=sum_rows, full_rows=full_rows)
    jobs = [("full", kt, it) for kt, it in sel] + [("rows", kt, it) for kt, it in positions]
    import multiprocessing as mp

    P, K, Sn, F = len(positions), len(sel), len(sum_rows), len(full_rows)
    out = dict(positions=np.array(positions), sum_rows=sum_rows, full_rows=full_rows,
               mesh_digest=R.mesh_digest(mesh.vertices, tris), sel_positions=np.array(sel).reshape(-1, 2),
               sum_cnt=np.zeros((P, Sn), np.int32), sum_hash=np.zeros((P, Sn), np.uint64),
               sum_abs=np.zeros((P, Sn)), sum_ax=np.zeros((P, Sn)), sum_max=np.zeros(P),
               sel_cnt=np.zeros((K, M), np.int32), sel_hash=np.zeros((K, M), np.uint64),
               sel_abs=np.zeros((K, M)), sel_ax=np.zeros((K, M)), sel_max=np.zeros(K))
    if c == 3:
        out["vertices"], out["triangles"] = mesh.vertices, tris
    pidx = {p: k for k, p in enumerate(positions)}
    sidx = {p: k for k, p in enumerate(sel)}
    ents = {}
    with mp.get_context("fork").Pool(args.workers) as pool:
        for n, (which, pos, st, ent, mx) in enumerate(pool.imap_unordered(_job, jobs)):
            if which == "rows":
                k = pidx[pos]
                out["sum_cnt"][k], out["sum_hash"][k], out["sum_abs"][k], out["sum_ax"][k] = st
                out["sum_max"][k] = mx
                ents[k] = ent
            else:
                k = sidx[pos]
                out["sel_cnt"][k], out["sel_hash"][k], out["sel_abs"][k], out["sel_ax"][k] = st
                out["sel_max"][k] = mx
            if n % 25 == 0:
                print(f"{n + 1}/{len(jobs)} {which} {pos} {time.time() - t0:.0f} s", flush=True)
    ind, dat, ptr = [], [], [0]
    for k in range(P):
        for cols, vals in ents[k]:
            ind.append(cols)
            dat.append(vals)
            ptr.append(ptr[-1] + len(cols))
    out["full_indptr"] = np.array(ptr, dtype=np.int64).reshape(-1)
    out["full_indices"] = np.concatenate(ind) if ind else np.zeros(0, np.int32)
    out["full_data"] = np.concatenate(dat) if dat else np.zeros(0)
    np.savez_compressed(os.path.join(OUT, f"blocks_cfg{c}.npz"), **out)
    print(f"wrote blocks_cfg{c}.npz in {time.time() - t0:.0f} s; entries {len(out['full_data'])}")


if __name__ == "__main__":
    main()
