"""ORACLE (baseline infrastructure): the REFERENCE package timed on the host cores.

Used only by bench.py (`--impl reference` and the cpu_baseline leg).  It never
imports the product package: mesh, grid, tables, positions, admissibility,
classification, rules, kernel and CSR build are all the reference's own
(`tdbem`, installed from /root/reference/pkg by `make -C oracle ref` into
oracle/_ref/pkg, or the driver's baseline/_ref).

One step = the reference's assemble_subblocks (ref/assembly.py:240-306) at EVERY
canonical block position (ref/block_system.py:249-263) for the test rows of a
seeded random sample of test vertices, positions spread over a fork pool of all
host cores (the reference's own parallelism is per position,
ref/block_system.py:259-263).  The mesh's distance bounds are pre-warmed before
the timed region, as the reference's CPU protocol prescribes (BASELINE.md 4.3,
SURVEY 8d): columns of the sampled test triangles only, from the reference's own
primitives in the reference's operation order (ref/mesh.py:357-391); every other
pair is inadmissible, so exactly the sampled rows' units are computed, plus the
touching pair of largest tmax per case (keeps the reference's n_rad,
ref/assembly.py:281-287).  value = admissible units computed / wall seconds.

Why a sample: the full reference assembly is ~1 h on 8 cores at config 4 and
infeasible at config 5 (SURVEY finding 8); a step of a few seconds keeps the
whole --steps/--warmup run within minutes.  The sampled estimator is calibrated
against full assemble_system runs at configs 1-2 (profiles/r02/).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

SPEC = {1: ("icosphere2_E320_dt0.1_N40", "ico", 2, 0.1, 40),
        2: ("icosphere3_E1280_dt0.05_N80", "ico", 3, 0.05, 80),
        3: ("cube16_E3072_dt0.05_N100", "cube", 0, 0.05, 100),
        4: ("icosphere4_E5120_dt0.025_N160", "ico", 4, 0.025, 160),
        5: ("icosphere5_E20480_dt0.025_N320", "ico", 5, 0.025, 320)}


def import_reference() -> str:
    """Put the installed reference package on sys.path; returns its location."""
    for d in (os.path.join(ROOT, "baseline", "_ref"), os.path.join(HERE, "_ref", "pkg")):
        if os.path.isfile(os.path.join(d, "tdbem", "__init__.py")):
            if d not in sys.path:
                sys.path.insert(0, d)
            import tdbem._kernels as K

            if K.backend_name != "compiled":
                raise RuntimeError(f"reference at {d} has no compiled kernel ({K.backend_name})")
            return d
    raise ImportError("reference package not installed (make -C oracle ref)")


def pair_bounds(corners, tris, ii, jj):
    """ref/mesh.py:357-391 op for op on an explicit pair list (reference primitives)."""
    from tdbem.mesh import point_triangle_distance, segment_segment_distance

    ca, cb = corners[ii], corners[jj]
    vdist = np.linalg.norm(ca[:, :, None, :] - cb[:, None, :, :], axis=3)
    dmax = vdist.max(axis=(1, 2))
    dmin = vdist.min(axis=(1, 2))
    for a in range(3):
        p0, p1 = ca[:, a], ca[:, (a + 1) % 3]
        for b in range(3):
            dmin = np.minimum(dmin, segment_segment_distance(p0, p1, cb[:, b], cb[:, (b + 1) % 3]))
    for a in range(3):
        dmin = np.minimum(dmin, point_triangle_distance(ca[:, a], cb[:, 0], cb[:, 1], cb[:, 2]))
        dmin = np.minimum(dmin, point_triangle_distance(cb[:, a], ca[:, 0], ca[:, 1], ca[:, 2]))
    shared = np.zeros(len(ii), dtype=bool)
    for a in range(3):
        for b in range(3):
            shared |= tris[ii, a] == tris[jj, b]
    dmin[shared] = 0.0
    return dmin, dmax


def config_inputs(c: int):
    from tdbem.mesh import SurfaceMesh, icosahedron, refine
    from tdbem.temporal_basis import TimeGrid

    name, kind, lv, dt, N = SPEC[c]
    if kind == "ico":
        m = icosahedron()
        for _ in range(lv):
            m = refine(m, project_unit_sphere=True)
    else:  # the committed jittered-cube arrays (the reference has no cube generator)
        g = np.load(os.path.join(ROOT, "tests", "golden", "blocks_cfg3.npz"))
        m = SurfaceMesh(g["vertices"], g["triangles"])
    return name, m, TimeGrid(T=float(f"{dt * (N - 1):.12g}"), N=N, p=0)


_W = {}


def _position(args):
    kt, it = args
    from tdbem.assembly import assemble_subblocks

    t0 = time.perf_counter()
    assemble_subblocks(_W["mesh"], _W["grid"], _W["tables"], kt, it)
    return (kt, it), time.perf_counter() - t0


class RowSampler:
    """Reference assembly of sampled test rows at every canonical position."""

    def __init__(self, c: int, rows_per_step: int, workers: int | None = None):
        self.where = import_reference()
        from tdbem.block_system import BlockHessenbergMatrix, canonical_position
        from tdbem.kernel_weights import is_zero_pair, psi_support, tables_for

        self.c = c
        self.name, self.mesh, self.grid = config_inputs(c)
        self.tables = tables_for(self.grid)
        g = self.grid
        A = BlockHessenbergMatrix(grid=g, M=self.mesh.num_vertices, diameter=self.mesh.diameter)
        pos = set()
        for kt in range(1, g.N + 1):
            for it in range(1, g.N + 1):
                if not A.is_zero_position(kt, it):
                    p = canonical_position(g, kt, it)
                    if p is not None:
                        pos.add(p)
        self.positions = sorted(pos)
        live = [p for p in self.positions if not is_zero_pair(g, *p)]
        sup = np.array([psi_support(g, *p) for p in live]).reshape(-1, 2)
        self.live, self.slo, self.shi = live, sup[:, 0], sup[:, 1]
        # heavier (small-lag, singular) positions first for load balance
        self.order = sorted(live, key=lambda p: sup[live.index(p), 0])
        self.rows_per_step = rows_per_step
        self.workers = workers or os.cpu_count() or 1
        tris = self.mesh.triangles
        E = self.mesh.num_triangles
        share = {}
        for e in range(E):
            for v in tris[e]:
                share.setdefault(int(v), []).append(e)
        cand = np.array(sorted({(a, b) for es in share.values() for a in es for b in es}))
        tmin, tmax = pair_bounds(self.mesh.corners, tris, cand[:, 0], cand[:, 1])
        nsh = (tris[cand[:, 0]][:, :, None] == tris[cand[:, 1]][:, None, :]).sum(axis=(1, 2))
        self.extra = []
        for ns in (3, 2, 1):
            m = np.flatnonzero(nsh == ns)
            k = m[np.argmax(tmax[m])]
            self.extra.append((int(cand[k, 0]), int(cand[k, 1]), tmin[k], tmax[k]))

    def prepare(self, seed: int):
        """Pre-warmed (untimed) row-restricted mesh for one step; returns its unit count."""
        from tdbem.mesh import SurfaceMesh

        mesh = self.mesh
        E, M = mesh.num_triangles, mesh.num_vertices
        tris = mesh.triangles
        rng = np.random.default_rng(10_000 + seed)
        rows = np.sort(rng.choice(M, self.rows_per_step, replace=False))
        S = np.flatnonzero(np.isin(tris, rows).any(axis=1))
        ii = np.repeat(np.arange(E), len(S))
        jj = np.tile(S, E)
        cmin, cmax = pair_bounds(mesh.corners, tris, ii, jj)
        rmin, rmax = pair_bounds(mesh.corners, tris, jj, ii)
        tmin = np.full((E, E), np.inf)
        tmax = np.full((E, E), -np.inf)
        tmin[ii, jj], tmax[ii, jj] = cmin, cmax
        for a, b, lo, hi in self.extra:
            tmin[a, b], tmax[a, b] = lo, hi
        both_min, both_max = tmin.copy(), tmax.copy()
        both_min[jj, ii], both_max[jj, ii] = rmin, rmax
        tmp = SurfaceMesh(mesh.vertices, tris)
        tmp.__dict__["tri_distance_bounds"] = (both_min, both_max)
        dof = type(mesh).dof_distance_bounds.func(tmp)
        R = SurfaceMesh(mesh.vertices, tris)
        R.__dict__["tri_distance_bounds"] = (tmin, tmax)
        R.__dict__["dof_distance_bounds"] = dof
        # admissible units of this restricted problem (what the step computes)
        ex = np.concatenate([ii, [e[0] for e in self.extra]])
        ey = np.concatenate([jj, [e[1] for e in self.extra]])
        lo, hi = tmin[ex, ey], tmax[ex, ey]
        units = int(sum(np.count_nonzero((lo <= b) & (hi >= a)) for a, b in zip(self.slo, self.shi)))
        return R, units, rows

    def step(self, prepared):
        """The timed part: reference assemble_subblocks of every position (fork pool)."""
        import multiprocessing as mp

        R, units, rows = prepared
        _W.update(mesh=R, grid=self.grid, tables=self.tables)
        t0 = time.perf_counter()
        with mp.get_context("fork").Pool(self.workers) as pool:
            list(pool.imap_unordered(_position, self.order, chunksize=1))
        return units, time.perf_counter() - t0

    def describe(self, steps: int) -> str:
        return (f"reference tdbem ({self.where}) assemble_subblocks at all {len(self.positions)} canonical "
                f"positions for the rows of {self.rows_per_step} seeded random test vertices per step "
                f"({steps} steps), fork pool of {self.workers} host processes; distance bounds pre-warmed "
                f"(untimed) for the sampled rows with the reference's primitives")


def full_units(c: int):
    """Total admissible units of config c from the reference-generated golden (units_cfg{c}.npz)."""
    path = os.path.join(ROOT, "tests", "golden", f"units_cfg{c}.npz")
    if not os.path.exists(path):
        return None, None
    g = np.load(path)
    return int(g["units"].sum()), len(g["positions"])


def available() -> bool:
    try:
        import_reference()
        return True
    except (ImportError, RuntimeError):
        return False

