"""ORACLE (test infrastructure): numpy restatement of the reference assembly path.

Follows, function by function (paths under /root/reference/pkg/src/tdbem/):
  segment_segment_distance   mesh.py:286-312
  _point_segment_distance    mesh.py:315-320
  point_triangle_distance    mesh.py:323-354
  tri_distance_bounds        mesh.py:146-153, _tri_pair_bounds :357-391 (chunked here)
  dof_distance_bounds        mesh.py:155-168
  block_pattern              assembly.py:167-184
  classify_pair              assembly.py:130-152
  _kahan_csr                 assembly.py:187-214
  _pair_group_values         assembly.py:217-237 (512-pair chunks)
  assemble_subblocks         assembly.py:240-306
  matvec                     block_system.py:180-216 (per-rank partial sums)
The hot kernel is oracle/pair_kernel.c (or the reference's own compiled
_core from oracle/_ref when built).  Inputs (mesh arrays, rules, tables) come
from the product's host modules, which are pinned bit-identical to the
reference by tests/test_host_golden.py.
"""

from __future__ import annotations

import ctypes as C
import importlib.util
import math
import os

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
_CHUNK = 512


# ---------------------------------------------------------------------------
# kernels: C restatement or the reference's own compiled _core
# ---------------------------------------------------------------------------
class _Pack(C.Structure):
    _fields_ = [
        ("p", C.c_int32), ("deg", C.c_int32), ("max_nsub", C.c_int32), ("reserved", C.c_int32),
        ("delta", C.c_double),
        ("lo", C.POINTER(C.c_double)), ("width", C.POINTER(C.c_double)),
        ("nsub", C.POINTER(C.c_int64)), ("coeffs", C.POINTER(C.c_double)),
        ("sp", C.POINTER(C.c_double)), ("sn", C.POINTER(C.c_double)),
        ("fold", C.POINTER(C.c_uint8)), ("active", C.POINTER(C.c_uint8)),
    ]


_LIB = None


def _oracle_lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.run(["make", "-C", HERE, "liboracle.so"], check=True, capture_output=True)
        lib = C.CDLL(path)
        D = C.POINTER(C.c_double)
        lib.oracle_pair_block_contributions.restype = C.c_int
        lib.oracle_pair_block_contributions.argtypes = [D] * 10 + [C.c_int64, C.c_int64, C.POINTER(_Pack), D]
        _LIB = lib
    return _LIB


def c_pair_block_contributions(cx, cy, a2x, a2y, ndot, curly, curlx, xhat, yhat, wq, pack):
    """Plain-C restatement of _core.pair_block_contributions (same contract)."""
    f = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    args = [f(a) for a in (cx, cy, a2x, a2y, ndot, curly, curlx, xhat, yhat, wq)]
    keep = dict(lo=f(pack.lo), width=f(pack.width), nsub=np.ascontiguousarray(pack.nsub, dtype=np.int64),
                coeffs=f(pack.coeffs), sp=f(pack.sp), sn=f(pack.sn),
                fold=np.ascontiguousarray(pack.fold, dtype=np.uint8),
                active=np.ascontiguousarray(pack.active, dtype=np.uint8))
    pk = _Pack()
    pk.p, pk.deg, pk.max_nsub = int(pack.p), keep["coeffs"].shape[2] - 1, keep["coeffs"].shape[1]
    pk.delta = float(pack.delta)
    D = C.POINTER(C.c_double)
    pk.lo, pk.width = keep["lo"].ctypes.data_as(D), keep["width"].ctypes.data_as(D)
    pk.nsub = keep["nsub"].ctypes.data_as(C.POINTER(C.c_int64))
    pk.coeffs = keep["coeffs"].ctypes.data_as(D)
    pk.sp, pk.sn = keep["sp"].ctypes.data_as(D), keep["sn"].ctypes.data_as(D)
    pk.fold = keep["fold"].ctypes.data_as(C.POINTER(C.c_uint8))
    pk.active = keep["active"].ctypes.data_as(C.POINTER(C.c_uint8))
    npair, nq = args[0].shape[0], args[9].shape[0]
    np1 = int(pack.p) + 1
    out = np.empty((npair, np1, np1, 3, 3))
    if npair:
        rc = _oracle_lib().oracle_pair_block_contributions(
            *[a.ctypes.data_as(D) for a in args], npair, nq, C.byref(pk), out.ctypes.data_as(D))
        if rc != 0:
            raise MemoryError("oracle kernel failed")
    return out


def ref_core():
    """The reference's own compiled kernel module (oracle/_ref), or None."""
    d = os.path.join(HERE, "_ref")
    if not os.path.isdir(d):
        return None
    for fn in os.listdir(d):
        if fn.startswith("_core") and fn.endswith(".so"):
            spec = importlib.util.spec_from_file_location("_core", os.path.join(d, fn))
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    return None


# ---------------------------------------------------------------------------
# distance bounds (mesh.py:286-391)
# ---------------------------------------------------------------------------
def segment_segment_distance(p0, p1, q0, q1):
    d1 = p1 - p0
    d2 = q1 - q0
    r = p0 - q0
    a = np.einsum("ij,ij->i", d1, d1)
    e = np.einsum("ij,ij->i", d2, d2)
    b = np.einsum("ij,ij->i", d1, d2)
    c = np.einsum("ij,ij->i", d1, r)
    f = np.einsum("ij,ij->i", d2, r)
    den = a * e - b * b
    a_s = np.where(a > 0, a, 1.0)
    e_s = np.where(e > 0, e, 1.0)
    s = np.where(den > 0.0, np.clip((b * f - c * e) / np.where(den > 0, den, 1.0), 0.0, 1.0), 0.0)
    t = (b * s + f) / e_s
    s = np.where(t < 0.0, np.clip(-c / a_s, 0.0, 1.0), s)
    s = np.where(t > 1.0, np.clip((b - c) / a_s, 0.0, 1.0), s)
    t = np.clip(t, 0.0, 1.0) * (e > 0.0)
    s = s * (a > 0.0)
    diff = p0 + s[:, None] * d1 - (q0 + t[:, None] * d2)
    return np.linalg.norm(diff, axis=1)


def _point_segment_distance(p, a, b):
    ab = b - a
    den = np.einsum("ij,ij->i", ab, ab)
    t = np.einsum("ij,ij->i", p - a, ab) / np.where(den > 0, den, 1.0)
    t = np.clip(t, 0.0, 1.0) * (den > 0.0)
    return np.linalg.norm(p - a - t[:, None] * ab, axis=1)


def point_triangle_distance(p, v0, v1, v2):
    e0 = v1 - v0
    e1 = v2 - v0
    n = np.cross(e0, e1)
    nn = np.einsum("ij,ij->i", n, n)
    w = p - v0
    dplane = np.abs(np.einsum("ij,ij->i", w, n)) / np.sqrt(np.where(nn > 0, nn, 1.0))
    d00 = np.einsum("ij,ij->i", e0, e0)
    d01 = np.einsum("ij,ij->i", e0, e1)
    d11 = np.einsum("ij,ij->i", e1, e1)
    d20 = np.einsum("ij,ij->i", w, e0)
    d21 = np.einsum("ij,ij->i", w, e1)
    den = d00 * d11 - d01 * d01
    den_s = np.where(den > 0, den, 1.0)
    u = (d11 * d20 - d01 * d21) / den_s
    v = (d00 * d21 - d01 * d20) / den_s
    inside = (u >= 0.0) & (v >= 0.0) & (u + v <= 1.0) & (den > 0.0) & (nn > 0.0)
    edge = np.minimum.reduce([
        _point_segment_distance(p, v0, v1),
        _point_segment_distance(p, v1, v2),
        _point_segment_distance(p, v2, v0),
    ])
    return np.where(inside, dplane, edge)


def tri_distance_bounds(mesh, rows=None):
    """(tmin, tmax) over triangle pairs [ex, ey] (rows = subset of ex, default all)."""
    corners, tris = mesh.corners, mesh.triangles
    E = len(corners)
    rows = np.arange(E) if rows is None else np.asarray(rows)
    tmin = np.empty((len(rows), E))
    tmax = np.empty((len(rows), E))
    step = max(1, 200000 // E)
    for r0 in range(0, len(rows), step):
        ri = rows[r0 : r0 + step]
        ii = np.repeat(ri, E)
        jj = np.tile(np.arange(E), len(ri))
        ca, cb = corners[ii], corners[jj]
        vd = np.linalg.norm(ca[:, :, None, :] - cb[:, None, :, :], axis=3)
        dmax = vd.max(axis=(1, 2))
        dmin = vd.min(axis=(1, 2))
        for a in range(3):
            for b in range(3):
                dmin = np.minimum(dmin, segment_segment_distance(ca[:, a], ca[:, (a + 1) % 3],
                                                                 cb[:, b], cb[:, (b + 1) % 3]))
        for a in range(3):
            dmin = np.minimum(dmin, point_triangle_distance(ca[:, a], cb[:, 0], cb[:, 1], cb[:, 2]))
            dmin = np.minimum(dmin, point_triangle_distance(cb[:, a], ca[:, 0], ca[:, 1], ca[:, 2]))
        shared = np.zeros(len(ii), dtype=bool)
        for a in range(3):
            for b in range(3):
                shared |= tris[ii, a] == tris[jj, b]
        dmin[shared] = 0.0
        tmin[r0 : r0 + len(ri)] = dmin.reshape(len(ri), E)
        tmax[r0 : r0 + len(ri)] = dmax.reshape(len(ri), E)
    return tmin, tmax


def dof_distance_bounds(mesh, tmin, tmax):
    m = mesh.num_vertices
    dmin = np.full((m, m), np.inf)
    dmax = np.zeros((m, m))
    t = mesh.triangles
    for a in range(3):
        for b in range(3):
            idx = (t[:, a][:, None], t[None, :, b])
            np.minimum.at(dmin, idx, tmin)
            np.maximum.at(dmax, idx, tmax)
    return dmin, dmax


# ---------------------------------------------------------------------------
# assembly (assembly.py:130-306)
# ---------------------------------------------------------------------------
def classify_pair(mesh, ex, ey):
    if ex == ey:
        return "coincident", (0, 1, 2), (0, 1, 2)
    tx, ty = mesh.triangles[ex], mesh.triangles[ey]
    shared = sorted(set(tx.tolist()) & set(ty.tolist()))
    if not shared:
        return "regular", (0, 1, 2), (0, 1, 2)

    def order(tri):
        lead = [int(np.flatnonzero(tri == g)[0]) for g in shared]
        return tuple(lead + [a for a in range(3) if a not in lead])

    return ("edge" if len(shared) == 2 else "vertex"), order(tx), order(ty)


def kahan_csr(rows, cols, vals, m):
    if len(vals) == 0:
        return sp.csr_matrix((m, m))
    key = rows.astype(np.int64) * m + cols
    order = np.argsort(key, kind="stable")
    key = key[order]
    vals = vals[order]
    starts = np.concatenate([[0], np.flatnonzero(np.diff(key)) + 1])
    seg = np.searchsorted(starts, np.arange(len(key)), side="right") - 1
    pos = np.arange(len(key)) - starts[seg]
    total = np.zeros(len(starts))
    comp = np.zeros(len(starts))
    for step in range(int(pos.max()) + 1):
        mk = pos == step
        s = seg[mk]
        y = vals[mk] - comp[s]
        t = total[s] + y
        comp[s] = (t - total[s]) - y
        total[s] = t
    ukey = key[starts]
    return sp.coo_matrix((total, (ukey // m, ukey % m)), shape=(m, m)).tocsr()


class OracleAssembler:
    """Reference-algorithm assembly on the CPU, one block position at a time."""

    def __init__(self, mesh, grid, tables, config=None, kernel="c", bounds=None):
        from paper_1503_07221_b200.assembly import QuadratureConfig

        self.mesh, self.grid, self.tables = mesh, grid, tables
        self.config = config or QuadratureConfig()
        if kernel == "c":
            self.kernel = c_pair_block_contributions
        elif kernel == "ref":
            core = ref_core()
            if core is None:
                raise RuntimeError("oracle/_ref not built (make -C oracle ref)")
            self.kernel = core.pair_block_contributions
        else:
            self.kernel = kernel
        self._bounds = bounds

    @property
    def bounds(self):
        if self._bounds is None:
            self._bounds = tri_distance_bounds(self.mesh)
        return self._bounds

    def pattern(self, kt, it):
        from paper_1503_07221_b200.kernel_weights import is_zero_pair, psi_support

        if is_zero_pair(self.grid, kt, it):
            return np.empty((0, 2), dtype=np.int64)
        slo, shi = psi_support(self.grid, kt, it)
        tmin, tmax = self.bounds
        ex, ey = np.nonzero((tmin <= shi) & (tmax >= slo))
        return np.column_stack([ex, ey]).astype(np.int64)

    def _group_values(self, pack, pairs, lx, ly, rule):
        m = self.mesh
        xhat, yhat, wq = rule
        ax = np.arange(len(pairs))
        cx = m.corners[pairs[:, 0]][ax[:, None], lx]
        cy = m.corners[pairs[:, 1]][ax[:, None], ly]
        a2x = 2.0 * m.areas[pairs[:, 0]]
        a2y = 2.0 * m.areas[pairs[:, 1]]
        ndot = np.einsum("pd,pd->p", m.normals[pairs[:, 0]], m.normals[pairs[:, 1]])
        curlx = m.curls[pairs[:, 0]][ax[:, None], lx]
        curly = m.curls[pairs[:, 1]][ax[:, None], ly]
        vals = []
        for c0 in range(0, len(pairs), _CHUNK):
            c1 = min(c0 + _CHUNK, len(pairs))
            vals.append(self.kernel(cx[c0:c1], cy[c0:c1], a2x[c0:c1], a2y[c0:c1], ndot[c0:c1],
                                    curly[c0:c1], curlx[c0:c1], xhat, yhat, wq, pack))
        return np.concatenate(vals)

    def subblocks(self, kt, it, with_units=False):
        from paper_1503_07221_b200.assembly import PsiPack
        from paper_1503_07221_b200.quadrature import pair_rule_regular, singular_rule

        mesh, grid, cfg = self.mesh, self.grid, self.config
        m = mesh.num_vertices
        np1 = grid.p + 1
        pairs = self.pattern(kt, it)
        empty = [[sp.csr_matrix((m, m)) for _ in range(np1)] for _ in range(np1)]
        if len(pairs) == 0:
            return (empty, 0) if with_units else empty
        pack = PsiPack.build(self.tables, grid, kt, it)
        groups = {"regular": [], "coincident": [], "edge": [], "vertex": []}
        for ex, ey in pairs:
            case, lx, ly = classify_pair(mesh, int(ex), int(ey))
            groups[case].append((int(ex), int(ey), lx, ly))
        vals_l, gx_l, gy_l = [], [], []
        for case in ("regular", "coincident", "edge", "vertex"):
            ent = groups[case]
            if not ent:
                continue
            parr = np.array([(e[0], e[1]) for e in ent], dtype=np.int64)
            lx = np.array([e[2] for e in ent], dtype=np.int64)
            ly = np.array([e[3] for e in ent], dtype=np.int64)
            if case == "regular":
                rule = pair_rule_regular(cfg.q_reg)
            else:
                n_rad = cfg.n_rad
                if n_rad is None:
                    rmax = float(self.bounds[1][parr[:, 0], parr[:, 1]].max())
                    n_rad = min(8, max(1, math.ceil(3.0 * rmax / grid.dt)))
                rule = singular_rule(case, cfg.q_sing, n_rad, 2 if n_rad > 1 else 1)
            vals_l.append(self._group_values(pack, parr, lx, ly, rule))
            ax = np.arange(len(parr))
            gx_l.append(mesh.triangles[parr[:, 0]][ax[:, None], lx])
            gy_l.append(mesh.triangles[parr[:, 1]][ax[:, None], ly])
        vals = np.concatenate(vals_l)
        gx = np.concatenate(gx_l)
        gy = np.concatenate(gy_l)
        rows = np.broadcast_to(gy[:, :, None], (len(gy), 3, 3)).reshape(-1)
        cols = np.broadcast_to(gx[:, None, :], (len(gx), 3, 3)).reshape(-1)
        out = [[kahan_csr(rows, cols, vals[:, m2, m1].reshape(-1), m) for m1 in range(np1)]
               for m2 in range(np1)]
        return (out, len(pairs)) if with_units else out


# ---------------------------------------------------------------------------
# block system + matvec (block_system.py)
# ---------------------------------------------------------------------------
def canonical_blocks(assembler, positions):
    """{(kt, it): nested CSR} for the given canonical positions."""
    return {pos: assembler.subblocks(*pos) for pos in positions}


def matvec(grid, M, diameter, blocks, x, rows=None, cols=None):
    """y = A x with the reference's resolve / sign / zero-position rules (block_system.py:180-216)."""
    from paper_1503_07221_b200.block_system import canonical_position, is_zero_position

    np1 = grid.p + 1
    rlo, rhi = rows if rows is not None else (1, grid.N)
    clo, chi = cols if cols is not None else (1, grid.N)
    y = np.zeros((rhi - rlo + 1) * np1 * M)
    inner = lambda t: 1 < t < grid.N
    for kt in range(rlo, rhi + 1):
        for it in range(clo, chi + 1):
            if is_zero_position(grid, diameter, kt, it):
                continue
            pos = canonical_position(grid, kt, it)
            stored = blocks.get(pos)
            if stored is None:
                continue
            for m2 in range(np1):
                r = ((kt - rlo) * np1 + m2) * M
                for m1 in range(np1):
                    c = ((it - clo) * np1 + m1) * M
                    if inner(kt) and inner(it) and m1 > m2:
                        blk, sgn = stored[m1][m2], float((-1) ** (m1 + m2))
                    else:
                        blk, sgn = stored[m2][m1], 1.0
                    y[r : r + M] += sgn * (blk @ x[c : c + M])
    return y


def dense(grid, M, diameter, blocks):
    n = grid.L * M
    out = np.zeros((n, n))
    eye = np.eye(n)
    for k in range(n):
        out[:, k] = matvec(grid, M, diameter, blocks, eye[:, k])
    return out


# ---------------------------------------------------------------------------
# right-hand side (assembly.py:314-355)
# ---------------------------------------------------------------------------
def assemble_rhs(mesh, grid, g, q_reg: int = 4):
    """Host restatement of the reference's load-vector loop (assembly.py:314-355),
    operation for operation (bit-identical, tests/test_oracle_golden.py)."""
    from paper_1503_07221_b200.quadrature import gauss_rule, triangle_rule
    from paper_1503_07221_b200.temporal_basis import basis_b, flat_index, support_interval

    m = mesh.num_vertices
    pts, w = triangle_rule(q_reg)
    c = mesh.corners
    X = (c[:, None, 0, :] + pts[None, :, 0, None] * (c[:, 1] - c[:, 0])[:, None, :]
         + pts[None, :, 1, None] * (c[:, 2] - c[:, 1])[:, None, :]).reshape(-1, 3)
    wx = (w[None, :] * 2.0 * mesh.areas[:, None]).reshape(-1)
    sh = np.column_stack([1.0 - pts[:, 0], pts[:, 0] - pts[:, 1], pts[:, 1]])
    dofs = np.repeat(mesh.triangles, len(pts), axis=0).reshape(-1)
    shw = np.tile(sh, (mesh.num_triangles, 1)) * wx[:, None]
    xg, wg = gauss_rule(2 * (grid.p + 4))
    out = np.zeros(grid.L * m)
    for k in range(1, grid.L + 1):
        idx = flat_index(grid, (k - 1) // (grid.p + 1) + 1, (k - 1) % (grid.p + 1))
        lo, hi = support_interval(grid, idx.timestep)
        nhalf = max(1, round((hi - lo) / (0.25 * grid.dt)))
        comp = np.zeros(m)
        for panel in range(nhalf):
            a = lo + (hi - lo) * panel / nhalf
            b = lo + (hi - lo) * (panel + 1) / nhalf
            tq = 0.5 * (a + b) + 0.5 * (b - a) * xg
            tw = 0.5 * (b - a) * wg * basis_b(grid, idx, tq, deriv=1)
            for ts, ws in zip(tq, tw):
                if ws == 0.0:
                    continue
                gv = np.asarray(g(X, ts), dtype=float)
                comp += np.bincount(dofs, weights=(shw * gv[:, None] * ws).reshape(-1), minlength=m)
        out[(k - 1) * m : k * m] = comp
    return out
