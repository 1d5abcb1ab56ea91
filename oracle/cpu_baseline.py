"""ORACLE (test / baseline infrastructure): CPU timing of the reference assembly path.

Used only by bench.py (cpu_baseline leg and --impl reference).  Times the
REFERENCE's own compiled hot kernel (oracle/_ref, built from
/root/reference/pkg/src/tdbem/_kernels/_core.pyx) or, when that is absent, the
C restatement (oracle/liboracle.so), driven the way assemble_subblocks drives it
(assembly.py:217-237: per block position and singular case, 512-pair chunks,
the same PsiPack and rules), on a stratified random sample of the workload's
units:

  * strata = pair case (regular, coincident, edge, vertex); the per-unit cost
    differs by ~250x between them (256 vs 60000 rule points);
  * in each stratum pairs are drawn uniformly and ALL their admissible
    positions are evaluated, so units/second of the stratum is a ratio
    estimator over units;
  * the full-workload CPU time is sum_c U_c / rate_c with the exact per-case
    unit counts U_c of the workload.

Excluded from the timed sample (reported, not hidden): the reference's O(E^2)
distance bounds (pre-warmed in the reference's own CPU protocol, BASELINE.md
4.3), classify_pair's Python loop and the Kahan CSR build (a few % of the
reference's assembly time).
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from . import assembly as OA

CASES = ("regular", "coincident", "edge", "vertex")


def pair_bounds(mesh, ex, ey):
    """tmin/tmax of explicit pairs (same primitives as OA.tri_distance_bounds)."""
    c, t = mesh.corners, mesh.triangles
    ca, cb = c[ex], c[ey]
    vd = np.linalg.norm(ca[:, :, None, :] - cb[:, None, :, :], axis=3)
    dmax = vd.max(axis=(1, 2))
    dmin = vd.min(axis=(1, 2))
    for a in range(3):
        for b in range(3):
            dmin = np.minimum(dmin, OA.segment_segment_distance(ca[:, a], ca[:, (a + 1) % 3],
                                                                cb[:, b], cb[:, (b + 1) % 3]))
    for a in range(3):
        dmin = np.minimum(dmin, OA.point_triangle_distance(ca[:, a], cb[:, 0], cb[:, 1], cb[:, 2]))
        dmin = np.minimum(dmin, OA.point_triangle_distance(cb[:, a], ca[:, 0], ca[:, 1], ca[:, 2]))
    shared = np.zeros(len(ex), dtype=bool)
    for a in range(3):
        for b in range(3):
            shared |= t[ex, a] == t[ey, b]
    dmin[shared] = 0.0
    return dmin, dmax


def kernel_by_name(kind: str):
    if kind == "reference":
        core = OA.ref_core()
        if core is None:
            raise RuntimeError("oracle/_ref is not built")
        return core.pair_block_contributions
    return OA.c_pair_block_contributions


def _sample_pairs(mesh, case, n, rng, touching):
    E = mesh.num_triangles
    if case != "regular":
        ex, ey, lx, ly = touching[case]
        if len(ex) == 0:
            return None
        idx = rng.choice(len(ex), size=min(n, len(ex)), replace=False)
        return ex[idx], ey[idx], lx[idx], ly[idx]
    tri = mesh.triangles
    out_x, out_y = [], []
    while len(out_x) < n:
        a = rng.integers(0, E, 4 * n)
        b = rng.integers(0, E, 4 * n)
        sh = np.zeros(len(a), dtype=bool)
        for i in range(3):
            for k in range(3):
                sh |= tri[a, i] == tri[b, k]
        keep = ~sh
        out_x.extend(a[keep].tolist())
        out_y.extend(b[keep].tolist())
    ex = np.array(out_x[:n], dtype=np.int64)
    ey = np.array(out_y[:n], dtype=np.int64)
    ident = np.tile(np.arange(3), (n, 1))
    return ex, ey, ident, ident


def build_tasks(mesh, grid, tables, plan, n_per_case, seed=0):
    """Per stratum: list of (rule, pack, chunk args) kernel calls covering the sampled units."""
    from paper_1503_07221_b200.assembly import PsiPack

    rng = np.random.default_rng(seed)
    from paper_1503_07221_b200.mesh import touching_pairs

    touching = touching_pairs(mesh)
    positions = [(kt, it, f.slo[s], f.shi[s]) for f in plan.families for s, (kt, it) in enumerate(f.positions)]
    packs = {}
    tasks = {}
    for case in CASES:
        smp = _sample_pairs(mesh, case, n_per_case[case], rng, touching)
        if smp is None:
            continue
        ex, ey, lx, ly = smp
        tmin, tmax = pair_bounds(mesh, ex, ey)
        rule = plan.rules[case]
        calls = []
        units = 0
        ax = np.arange(len(ex))
        cx = mesh.corners[ex][ax[:, None], lx]
        cy = mesh.corners[ey][ax[:, None], ly]
        a2x, a2y = 2.0 * mesh.areas[ex], 2.0 * mesh.areas[ey]
        nd = np.einsum("pd,pd->p", mesh.normals[ex], mesh.normals[ey])
        curlx = mesh.curls[ex][ax[:, None], lx]
        curly = mesh.curls[ey][ax[:, None], ly]
        for kt, it, slo, shi in positions:
            adm = np.flatnonzero((tmin <= shi) & (tmax >= slo))
            if len(adm) == 0:
                continue
            if (kt, it) not in packs:
                packs[(kt, it)] = PsiPack.build(tables, grid, kt, it)
            units += len(adm)
            step = 512 if case == "regular" else 1  # singular: one pair per call (load balance)
            for c0 in range(0, len(adm), step):
                sel = adm[c0 : c0 + step]
                calls.append((cx[sel], cy[sel], a2x[sel], a2y[sel], nd[sel], curly[sel], curlx[sel],
                              rule[0], rule[1], rule[2], packs[(kt, it)]))
        tasks[case] = (units, calls)
    return tasks


def _run_calls(args):
    kind, calls = args
    k = kernel_by_name(kind)
    t0 = time.perf_counter()
    for c in calls:
        k(*c)
    return time.perf_counter() - t0


def measure(tasks, kind="reference", workers=1):
    """{case: (units, seconds)}: seconds = wall time of the stratum's calls on `workers` processes."""
    out = {}
    if workers <= 1:
        for case, (units, calls) in tasks.items():
            out[case] = (units, _run_calls((kind, calls)))
        return out
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        for case, (units, calls) in tasks.items():
            # split calls round-robin; wall time of the slowest shard
            shards = [(kind, calls[i::workers]) for i in range(workers)]
            t0 = time.perf_counter()
            pool.map(_run_calls, shards, chunksize=1)
            out[case] = (units, time.perf_counter() - t0)
    return out


def estimate(measured, units_case):
    """Full-workload seconds and units/s from per-stratum rates and exact stratum sizes."""
    total_units = sum(units_case.values())
    seconds = 0.0
    for case, U in units_case.items():
        if U == 0:
            continue
        u, t = measured[case]
        seconds += U * (t / max(u, 1))
    return seconds, (total_units / seconds if seconds > 0 else float("nan"))


def default_sample(units_case, target_seconds=8.0, cost_hint=None):
    """Pairs per stratum so the sample costs roughly target_seconds on one core."""
    return {"regular": 400, "coincident": 4, "edge": 4, "vertex": 6}
