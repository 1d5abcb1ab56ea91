"""Galerkin assembly of block positions on the GPU (host orchestration).

Reference interface (``tdbem.assembly``, /root/reference/pkg/src/tdbem/assembly.py):
  QuadratureConfig      :52-65
  PsiPack / .build      :68-127
  classify_pair         :130-152
  assemble_subblocks    :240-306   -> device all-lags assembly of one position
  assemble_block        :309-311
Entries are
    (n_x.n_y)/(4 pi |x-y|) phi_j(y) phi_l(x) psi(|x-y|)
  + (curl phi_j(y) . curl phi_l(x))/(4 pi |x-y|) psi~(|x-y|)
rows j = y (test) vertex, columns l = x (ansatz) vertex.

All quadrature runs in libtdb.so (csrc/tdb_assembly.cu); this module only
builds the small host-side plan (positions grouped into table families, the
reference rules, n_rad) and converts device CSR to scipy on request.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .kernel_weights import PrototypeTables, is_zero_pair, psi_support, tables_for
from .mesh import SurfaceMesh, touching_pairs
from .quadrature import Q_REG, Q_SING, n_rad_for, pair_rule_regular, singular_rule
from .temporal_basis import TimeGrid, canonical_origin, timestep_kind

__all__ = [
    "QuadratureConfig",
    "PsiPack",
    "classify_pair",
    "assemble_subblocks",
    "assemble_block",
    "AssemblyPlan",
    "build_plan",
    "DeviceAssembly",
]

CASES = ("regular", "coincident", "edge", "vertex")


@dataclass(frozen=True)
class QuadratureConfig:
    """q_reg x q_reg collapsed Gauss per triangle for separated pairs; q_sing
    tensor Gauss with n_rad x n_ang panels for touching pairs (n_rad=None:
    min(8, ceil(3 rmax/dt)) from the touching pairs' largest corner distance)."""

    q_reg: int = Q_REG
    q_sing: int = Q_SING
    n_rad: int | None = None


@dataclass
class PsiPack:
    """Packed tables of one block position; t = (m2 (p+1) + m1) * 2 + {0: psi, 1: psi~}."""

    p: int
    delta: float
    lo: np.ndarray
    width: np.ndarray
    nsub: np.ndarray
    coeffs: np.ndarray
    sp: np.ndarray
    sn: np.ndarray
    fold: np.ndarray
    active: np.ndarray

    @classmethod
    def build(cls, tables: PrototypeTables, grid: TimeGrid, kt: int, it: int) -> "PsiPack":
        p = grid.p
        ki, kk = timestep_kind(grid, it), timestep_kind(grid, kt)
        nt = 2 * (p + 1) ** 2
        entries = []
        for m2 in range(p + 1):
            for m1 in range(p + 1):
                for tilde in (False, True):
                    entries.append(tables.resolve(tilde, ki, kk, m1, m2))
        max_nsub = max([1] + [e[0].n_sub for e in entries if e[0] is not None])
        pack = cls(
            p=p,
            delta=canonical_origin(grid, it) - canonical_origin(grid, kt),
            lo=np.zeros(nt), width=np.ones(nt), nsub=np.ones(nt, dtype=np.int64),
            coeffs=np.zeros((nt, max_nsub, tables.deg + 1)),
            sp=np.ones(nt), sn=np.ones(nt),
            fold=np.zeros(nt, dtype=np.uint8), active=np.zeros(nt, dtype=np.uint8),
        )
        for t, (tbl, s_pos, s_neg, fold) in enumerate(entries):
            if tbl is None:
                continue
            pack.active[t] = 1
            pack.lo[t], pack.width[t], pack.nsub[t] = tbl.lo, tbl.width, tbl.n_sub
            pack.coeffs[t, : tbl.n_sub] = tbl.coeffs
            pack.sp[t], pack.sn[t] = s_pos, s_neg
            pack.fold[t] = 1 if fold else 0
        return pack

    def to_c(self, keep: list) -> _lib.TdbPsiPack:
        """C view of the pack; arrays appended to `keep` stay alive with it."""
        arrs = dict(
            lo=_lib.f64(self.lo), width=_lib.f64(self.width),
            nsub=np.ascontiguousarray(self.nsub, dtype=np.int64),
            coeffs=_lib.f64(self.coeffs), sp=_lib.f64(self.sp), sn=_lib.f64(self.sn),
            fold=np.ascontiguousarray(self.fold, dtype=np.uint8),
            active=np.ascontiguousarray(self.active, dtype=np.uint8),
        )
        keep.append(arrs)
        c = _lib.TdbPsiPack()
        c.p = self.p
        c.deg = arrs["coeffs"].shape[2] - 1
        c.max_nsub = arrs["coeffs"].shape[1]
        c.delta = float(self.delta)
        c.lo, c.width = _lib.ptr(arrs["lo"]), _lib.ptr(arrs["width"])
        c.nsub = _lib.ptr(arrs["nsub"], _lib.C.c_int64)
        c.coeffs = _lib.ptr(arrs["coeffs"])
        c.sp, c.sn = _lib.ptr(arrs["sp"]), _lib.ptr(arrs["sn"])
        c.fold = _lib.ptr(arrs["fold"], _lib.C.c_uint8)
        c.active = _lib.ptr(arrs["active"], _lib.C.c_uint8)
        return c


def classify_pair(mesh: SurfaceMesh, ex: int, ey: int):
    """(case, lx, ly): shared vertices first in ascending global order."""
    if ex == ey:
        return "coincident", (0, 1, 2), (0, 1, 2)
    tx = [int(v) for v in mesh.triangles[ex]]
    ty = [int(v) for v in mesh.triangles[ey]]
    shared = sorted(set(tx) & set(ty))
    if not shared:
        return "regular", (0, 1, 2), (0, 1, 2)

    def lead(t):
        first = [t.index(g) for g in shared]
        return tuple(first + [a for a in range(3) if a not in first])

    return ("edge" if len(shared) == 2 else "vertex"), lead(tx), lead(ty)


# ---------------------------------------------------------------------------
# plan: positions grouped into table families
# ---------------------------------------------------------------------------
@dataclass
class Family:
    kinds: tuple          # (kind_i, kind_k)
    positions: list       # [(kt, it)] in lag order
    delta: np.ndarray
    slo: np.ndarray
    shi: np.ndarray
    pack: PsiPack


@dataclass
class AssemblyPlan:
    grid: TimeGrid
    families: list
    where: dict           # (kt, it) -> (family index, s)
    rules: dict           # case -> (xhat, yhat, w)
    n_rad: dict           # case -> n_rad used


def _touching_tmax(mesh: SurfaceMesh):
    """Largest corner distance of every touching pair, per case (mesh.py:366-369).

    Mesh-derived, so it is cached on the mesh object (the reference caches its
    distance bounds on the mesh the same way, mesh.py:146-153)."""
    cached = getattr(mesh, "_tdb_touching_tmax", None)
    if cached is not None:
        return cached
    out = {}
    for case, (ex, ey, _, _) in touching_pairs(mesh).items():
        if len(ex) == 0:
            out[case] = np.zeros(0)
            continue
        diff = mesh.corners[ex][:, :, None, :] - mesh.corners[ey][:, None, :, :]
        out[case] = np.linalg.norm(diff, axis=3).max(axis=(1, 2))
    try:
        object.__setattr__(mesh, "_tdb_touching_tmax", out)  # frozen dataclass: like cached_property
    except (AttributeError, TypeError):
        pass
    return out


def build_plan(mesh: SurfaceMesh, grid: TimeGrid, tables: PrototypeTables, positions,
               config: QuadratureConfig = QuadratureConfig()) -> AssemblyPlan:
    groups: dict = {}
    for kt, it in positions:
        if is_zero_pair(grid, kt, it):
            continue
        key = (timestep_kind(grid, it), timestep_kind(grid, kt))
        groups.setdefault(key, []).append((kt, it))
    families = []
    where = {}
    for key in sorted(groups):
        pos = groups[key]
        d = np.array([canonical_origin(grid, it) - canonical_origin(grid, kt) for kt, it in pos])
        order = np.argsort(-d, kind="stable")
        pos = [pos[i] for i in order]
        sup = np.array([psi_support(grid, kt, it) for kt, it in pos]).reshape(-1, 2)
        slo, shi = sup[:, 0].copy(), sup[:, 1].copy()
        if np.any(np.diff(slo) < 0) or np.any(np.diff(shi) < 0):
            raise AssertionError(f"family {key}: supports not monotone in lag order")
        pack = PsiPack.build(tables, grid, pos[0][0], pos[0][1])
        if not np.all(pack.active):
            continue  # unreachable variant (e.g. last/first): identically zero
        f = len(families)
        families.append(Family(key, pos, d[order], slo, shi, pack))
        for s, ktit in enumerate(pos):
            where[ktit] = (f, s)

    rules = {"regular": pair_rule_regular(config.q_reg)}
    n_rad = {}
    tmax = _touching_tmax(mesh) if families else {}
    all_slo = np.concatenate([f.slo for f in families]) if families else np.zeros(0)
    for case in CASES[1:]:
        if config.n_rad is not None:
            nr = config.n_rad
        else:
            tm = tmax.get(case, np.zeros(0))
            vals = set()
            # rmax of the case at every position where any pair of it is admissible
            # (touching pairs have tmin = 0, so admissible iff slo <= tmax)
            for s in np.unique(all_slo):
                adm = tm[tm >= s]
                if len(adm):
                    vals.add(n_rad_for(float(adm.max()), grid.dt))
            if len(vals) > 1:
                raise NotImplementedError(f"{case}: n_rad varies across positions {vals}")
            nr = vals.pop() if vals else 1
        n_rad[case] = nr
        rules[case] = singular_rule(case, config.q_sing, nr, 2 if nr > 1 else 1)
    return AssemblyPlan(grid, families, where, rules, n_rad)


def _mesh_c(mesh: SurfaceMesh, keep: list) -> _lib.TdbMesh:
    off, ids = mesh.star_csr
    arrs = dict(
        corners=_lib.f64(mesh.corners), a2=_lib.f64(2.0 * mesh.areas), normals=_lib.f64(mesh.normals),
        curls=_lib.f64(mesh.curls), tri=np.ascontiguousarray(mesh.triangles, dtype=np.int64),
        off=np.ascontiguousarray(off, dtype=np.int64), ids=np.ascontiguousarray(ids, dtype=np.int64),
    )
    keep.append(arrs)
    m = _lib.TdbMesh()
    m.num_vertices, m.num_triangles = mesh.num_vertices, mesh.num_triangles
    m.corners, m.a2 = _lib.ptr(arrs["corners"]), _lib.ptr(arrs["a2"])
    m.normals, m.curls = _lib.ptr(arrs["normals"]), _lib.ptr(arrs["curls"])
    I64 = _lib.C.c_int64
    m.triangles = _lib.ptr(arrs["tri"], I64)
    m.star_off = _lib.ptr(arrs["off"], I64)
    m.star_ids = _lib.ptr(arrs["ids"], I64)
    return m


def _host_empty(shape, dtype):
    """Host array for device->host copies: page-locked memory from torch's caching
    host allocator (DMA at full PCIe/C2C speed, no first-touch page faults; blocks
    are recycled once the caller drops the array).  numpy fallback without CUDA."""
    try:
        import torch

        if torch.cuda.is_available():
            t = torch.empty(int(np.prod(shape)), dtype=getattr(torch, np.dtype(dtype).name), pin_memory=True)
            return t.numpy().reshape(shape)
    except (ImportError, RuntimeError, AttributeError):
        pass
    return np.empty(shape, dtype=dtype)


class DeviceAssembly:
    """Owner of a device-resident assembled system (TdbSystem handle).

    rows: optional strictly increasing test-vertex ids (a multi-GPU row block);
    only those CSR rows are assembled, from the pairs whose test triangle lies in
    their stars.  Default: every vertex.
    """

    def __init__(self, mesh: SurfaceMesh, plan: AssemblyPlan, ctx: _lib.Context | None = None, rows=None,
                 create_only: bool = False):
        self.mesh = mesh
        self.plan = plan
        self.ctx = ctx or _lib.default_context()
        self.M = mesh.num_vertices
        self.p = plan.grid.p
        self.handle = None
        self.rows = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
        self.nrows = self.M if self.rows is None else len(self.rows)
        keep: list = []
        fams = (_lib.TdbFamily * max(1, len(plan.families)))()
        for i, f in enumerate(plan.families):
            arr = dict(delta=_lib.f64(f.delta), slo=_lib.f64(f.slo), shi=_lib.f64(f.shi))
            keep.append(arr)
            fams[i].npos = len(f.positions)
            fams[i].delta, fams[i].slo, fams[i].shi = (_lib.ptr(arr[k]) for k in ("delta", "slo", "shi"))
            fams[i].pack = f.pack.to_c(keep)
        desc = _lib.TdbAssemblyDesc()
        desc.p = self.p
        desc.num_families = len(plan.families)
        desc.families = fams
        for c, case in enumerate(CASES):
            xh, yh, w = (_lib.f64(a) for a in plan.rules[case])
            keep.append((xh, yh, w))
            desc.rules[c].nq = len(w)
            desc.rules[c].xhat, desc.rules[c].yhat, desc.rules[c].w = _lib.ptr(xh), _lib.ptr(yh), _lib.ptr(w)
        if self.rows is not None:
            desc.num_rows = len(self.rows)
            desc.rows = _lib.ptr(self.rows, _lib.C.c_int64)
        self.num_families = len(plan.families)
        if self.num_families == 0:
            return
        h = _lib.C.c_void_p()
        fn = _lib.LIB.tdb_system_create if create_only else _lib.LIB.tdb_system_assemble
        _lib.check(fn(self.ctx.handle, _lib.C.byref(_mesh_c(mesh, keep)), _lib.C.byref(desc), _lib.C.byref(h)),
                   "system_assemble")
        self.handle = h

    def rerun(self) -> None:
        """Recompute every block from the device-resident inputs (no host round trips)."""
        if self.handle is not None:
            _lib.check(_lib.LIB.tdb_system_run(self.handle), "system_run")

    def stats(self) -> dict:
        if self.handle is None:
            return {}
        st = _lib.TdbStats()
        _lib.check(_lib.LIB.tdb_system_stats(self.handle, _lib.C.byref(st)), "system_stats")
        return st.as_dict()

    def family_arrays(self, f: int):
        """(indptr (npos*M+1,), indices (nnz,), data (nnz, (p+1)^2)) of family f on the host."""
        nnz = _lib.C.c_int64()
        _lib.check(_lib.LIB.tdb_system_family_nnz(self.handle, f, _lib.C.byref(nnz)), "family_nnz")
        npos = len(self.plan.families[f].positions)
        indptr = _host_empty((npos * self.nrows + 1,), np.int64)
        indices = _host_empty((max(1, nnz.value),), np.int32)
        data = _host_empty((max(1, nnz.value), (self.p + 1) ** 2), np.float64)
        _lib.check(_lib.LIB.tdb_system_copy_family(
            self.handle, f, _lib.ptr(indptr, _lib.C.c_int64), _lib.ptr(indices, _lib.C.c_int32),
            _lib.ptr(data)), "copy_family")
        return indptr, indices[: nnz.value], data[: nnz.value]

    def position_units(self) -> dict:
        """(kt, it) -> admissible-pair count of every assembled position (block_pattern size,
        ref/assembly.py:167-184) over this system's test triangles."""
        out = {}
        for f, fam in enumerate(self.plan.families):
            if self.handle is None:
                break
            u = np.zeros(len(fam.positions), dtype=np.int64)
            _lib.check(_lib.LIB.tdb_system_position_units(self.handle, f, _lib.ptr(u, _lib.C.c_int64)),
                       "position_units")
            out.update({pos: int(u[s]) for s, pos in enumerate(fam.positions)})
        return out

    def family_splits(self) -> dict:
        """(ansatz kind, test kind) -> (R, D, K) evaluation split of each family (tdb_system_family_split)."""
        out = {}
        for f, fam in enumerate(self.plan.families):
            if self.handle is None:
                break
            R, D, K = (_lib.C.c_int32() for _ in range(3))
            _lib.check(_lib.LIB.tdb_system_family_split(self.handle, f, _lib.C.byref(R), _lib.C.byref(D),
                                                        _lib.C.byref(K)), "family_split")
            out[tuple(fam.kinds)] = (R.value, D.value, K.value)
        return out

    def family_device(self, f: int):
        a, b, c = _lib.C.c_void_p(), _lib.C.c_void_p(), _lib.C.c_void_p()
        _lib.check(_lib.LIB.tdb_system_family_device(self.handle, f, _lib.C.byref(a), _lib.C.byref(b),
                                                     _lib.C.byref(c)), "family_device")
        return a.value, b.value, c.value

    def position_blocks(self, kt: int, it: int, _cache: dict | None = None):
        """Nested (p+1) x (p+1) list of scipy CSR blocks of position (kt, it)."""
        np1 = self.p + 1
        m = self.M
        loc = self.plan.where.get((kt, it))
        if loc is None or self.handle is None:
            return [[sp.csr_matrix((m, m)) for _ in range(np1)] for _ in range(np1)]
        f, s = loc
        if _cache is not None and f in _cache:
            indptr, indices, data = _cache[f]
        else:
            indptr, indices, data = self.family_arrays(f)
            if _cache is not None:
                _cache[f] = (indptr, indices, data)
        nr = self.nrows
        lo, hi = indptr[s * nr], indptr[(s + 1) * nr]
        ipl = indptr[s * nr : (s + 1) * nr + 1] - lo
        if self.rows is None:
            ip = ipl
        else:  # owned rows only: expand the local row pointer to all M rows
            counts = np.zeros(m, dtype=np.int64)
            counts[self.rows] = np.diff(ipl)
            ip = np.concatenate([[0], np.cumsum(counts)])
        out = []
        for m2 in range(np1):
            row = []
            for m1 in range(np1):
                vals = data[lo:hi, m2 * np1 + m1].copy()
                row.append(sp.csr_matrix((vals, indices[lo:hi].copy(), ip.copy()), shape=(m, m)))
            out.append(row)
        return out

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib.LIB is not None:  # LIB is None at interpreter exit
            _lib.LIB.tdb_system_destroy(h)
            self.handle = None


def as_product_inputs(mesh, grid):
    """Accept the reference's SurfaceMesh / TimeGrid (or any look-alike) as well as ours."""
    if not isinstance(mesh, SurfaceMesh):
        mesh = SurfaceMesh(np.asarray(mesh.vertices), np.asarray(mesh.triangles))
    if not isinstance(grid, TimeGrid):
        grid = TimeGrid(T=float(grid.T), N=int(grid.N), p=int(grid.p))
    return mesh, grid


def _as_tables(tables, grid):
    """Reference PrototypeTables work as-is (same attributes); None -> our cache."""
    return tables_for(grid) if tables is None else tables


def assemble_subblocks(mesh: SurfaceMesh, grid: TimeGrid, tables: PrototypeTables, kt: int, it: int,
                       config: QuadratureConfig = QuadratureConfig()):
    """All (p+1) x (p+1) CSR sub-blocks of block position (kt, it) (device assembly)."""
    mesh, grid = as_product_inputs(mesh, grid)
    tables = _as_tables(tables, grid)
    plan = build_plan(mesh, grid, tables, [(kt, it)], config)
    dev = DeviceAssembly(mesh, plan)
    return dev.position_blocks(kt, it)


def assemble_block(mesh, grid, tables, kt, it, m2, m1, config=QuadratureConfig()):
    return assemble_subblocks(mesh, grid, tables, kt, it, config)[m2][m1]


def tri_distance_bounds(mesh: SurfaceMesh, rows=None, ctx: _lib.Context | None = None):
    """Device drop-in for SurfaceMesh.tri_distance_bounds (mesh.py:146-153):
    (tmin, tmax) of triangle rows x all triangles, bit-identical to the reference."""
    ctx = ctx or _lib.default_context()
    E = mesh.num_triangles
    rows = np.arange(E, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    tmin = np.empty((len(rows), E))
    tmax = np.empty((len(rows), E))
    keep: list = []
    _lib.check(_lib.LIB.tdb_tri_distance_bounds(
        ctx.handle, _lib.C.byref(_mesh_c(mesh, keep)), len(rows), _lib.ptr(rows, _lib.C.c_int64),
        _lib.ptr(tmin), _lib.ptr(tmax)), "tri_distance_bounds")
    return tmin, tmax


def assemble_rhs(mesh: SurfaceMesh, grid: TimeGrid, g, config: QuadratureConfig = QuadratureConfig()):
    """Load vector b[(k-1) M + l] = int int g(x, t) phi_l(x) bdot_k(t) dx dt, on the GPU.

    Replaces assembly.py:314-355 of the reference: regular q_reg triangle rule in
    space; in time, Gauss panels of 2(p+4) points over quarter steps of each basis
    function's support (nodes and weights built on the host in the reference's
    arithmetic).  The datum is evaluated at every (time node, rule point):
      * g.device_eval(X, t) (torch tensors: X (P, 3), t (n,) -> (n, P)) on the GPU when
        the datum provides it (gaussian_pulse_neumann does);
      * otherwise g(X, t) -> (P,) is the reference's host callback contract (numpy),
        called per time node on the host and uploaded in chunks.
    The vertex gather and the per-basis time sum run in csrc/tdb_rhs.cu.  There is no
    CPU fallback: without a CUDA device this raises (the host restatement of the
    reference loop is the oracle's, oracle/assembly.py assemble_rhs).
    """
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("assemble_rhs: no CUDA device (the product has no CPU path)")
    return _assemble_rhs_device(mesh, grid, g, config)


def _rhs_time_nodes(grid: TimeGrid):
    """Time nodes / weights of every basis function, in the reference's arithmetic
    (assembly.py:339-349): (kptr (L+1,), t (n,), w (n,)); zero weights are kept."""
    from .quadrature import gauss_rule
    from .temporal_basis import basis_b, flat_index, support_interval

    xg, wg = gauss_rule(2 * (grid.p + 4))
    ts, ws, kptr = [], [], [0]
    for k in range(1, grid.L + 1):
        idx = flat_index(grid, (k - 1) // (grid.p + 1) + 1, (k - 1) % (grid.p + 1))
        lo, hi = support_interval(grid, idx.timestep)
        nhalf = max(1, round((hi - lo) / (0.25 * grid.dt)))
        for panel in range(nhalf):
            a = lo + (hi - lo) * panel / nhalf
            b = lo + (hi - lo) * (panel + 1) / nhalf
            tq = 0.5 * (a + b) + 0.5 * (b - a) * xg
            ts.append(tq)
            ws.append(0.5 * (b - a) * wg * basis_b(grid, idx, tq, deriv=1))
        kptr.append(kptr[-1] + nhalf * len(xg))
    return np.asarray(kptr, dtype=np.int64), np.concatenate(ts), np.concatenate(ws)


def _assemble_rhs_device(mesh: SurfaceMesh, grid: TimeGrid, g, config: QuadratureConfig = QuadratureConfig()):
    """assemble_rhs on the GPU: the datum at every (time node, rule point) in node
    chunks (device_eval on the GPU, or the host callback per node), vertex gather +
    per-basis time sum in csrc/tdb_rhs.cu."""
    import ctypes

    import torch

    from .quadrature import triangle_rule

    mesh, grid = as_product_inputs(mesh, grid)
    dev = torch.device("cuda", torch.cuda.current_device())
    m = mesh.num_vertices
    pts, w = triangle_rule(config.q_reg)
    c = mesh.corners
    X = (c[:, None, 0, :] + pts[None, :, 0, None] * (c[:, 1] - c[:, 0])[:, None, :]
         + pts[None, :, 1, None] * (c[:, 2] - c[:, 1])[:, None, :]).reshape(-1, 3)
    wx = (w[None, :] * 2.0 * mesh.areas[:, None]).reshape(-1)
    sh = np.column_stack([1.0 - pts[:, 0], pts[:, 0] - pts[:, 1], pts[:, 1]])
    shw = np.tile(sh, (mesh.num_triangles, 1)) * wx[:, None]          # (P, 3)
    dofs = np.repeat(mesh.triangles, len(pts), axis=0)                # (P, 3)
    P = len(X)
    # vertex -> (rule point, weight) CSR, points ascending (element order)
    vert = dofs.reshape(-1)
    order = np.argsort(vert, kind="stable")
    vptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(vptr, vert + 1, 1)
    vptr = np.cumsum(vptr)
    vpts = (order // 3).astype(np.int32)
    vw = shw.reshape(-1)[order]
    kptr, ts, ws = _rhs_time_nodes(grid)
    nn = len(ts)
    T = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    Xd, vptr_d, vpts_d, vw_d = T(X), T(vptr, torch.int64), T(vpts, torch.int32), T(vw)
    ts_d, ws_d, kptr_d = T(ts), T(ws), T(kptr, torch.int64)
    H = torch.empty((nn, m), dtype=torch.float64, device=dev)
    out = torch.empty(grid.L * m, dtype=torch.float64, device=dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    chunk = max(1, min(nn, (1 << 27) // max(P, 1)))  # <= 1 GiB of datum values per chunk
    for j0 in range(0, nn, chunk):
        nj = min(chunk, nn - j0)
        if hasattr(g, "device_eval"):
            G = g.device_eval(Xd, ts_d[j0 : j0 + nj]).to(torch.float64).contiguous()
        else:  # host callback g(X, t) -> (P,), the reference's contract (assembly.py:326)
            Gh = np.empty((nj, P))
            for i in range(nj):
                Gh[i] = np.asarray(g(X, float(ts[j0 + i])), dtype=float)
            G = torch.as_tensor(Gh).to(dev)
        _lib.check(_lib.LIB.tdb_rhs_vertex_gather(p(G), j0, nj, P, p(vptr_d), p(vpts_d), p(vw_d), m, p(H), stream),
                   "rhs_vertex_gather")
    _lib.check(_lib.LIB.tdb_rhs_time_sum(p(H), p(kptr_d), p(ws_d), grid.L, m, p(out), stream), "rhs_time_sum")
    return out.cpu().numpy()


class GaussianPulseNeumann:
    """g = -d_n u_inc for u_inc = f(t - t0 - (z - z_min)), f(s) = exp(-s^2/(2 sigma^2))
    (plane wave along +z with a Gaussian envelope; g = n_z f'(s)).
    Points are the triangle-rule points in element order, as assemble_rhs passes them.
    Callable on numpy arrays (host, the reference's callback contract) and, through
    device_eval, on CUDA tensors for a whole batch of times."""

    def __init__(self, mesh: SurfaceMesh, sigma: float = 0.2, t0: float = 1.0):
        self.zmin = float(mesh.vertices[:, 2].min())
        self.nz = mesh.normals[:, 2]
        self.E = mesh.num_triangles
        self.sigma, self.t0 = sigma, t0
        self._nz_dev = None

    def __call__(self, X, t):
        nq = len(X) // self.E
        sigma = self.sigma
        s = t - self.t0 - (X[:, 2] - self.zmin)
        f = np.exp(-s * s / (2.0 * sigma * sigma))
        return np.repeat(self.nz, nq) * (-s / sigma**2) * f

    def device_eval(self, X, t):
        import torch

        nq = X.shape[0] // self.E
        if self._nz_dev is None or self._nz_dev.device != X.device or self._nz_dev.numel() != X.shape[0]:
            self._nz_dev = torch.as_tensor(np.repeat(self.nz, nq)).to(X.device)
        sigma = self.sigma
        s = t[:, None] - self.t0 - (X[None, :, 2] - self.zmin)
        f = torch.exp(-s * s / (2.0 * sigma * sigma))
        return self._nz_dev[None, :] * (-s / sigma**2) * f


def gaussian_pulse_neumann(mesh: SurfaceMesh, sigma: float = 0.2, t0: float = 1.0):
    """The benchmark datum (SURVEY 8d RHS) as a GaussianPulseNeumann."""
    return GaussianPulseNeumann(mesh, sigma, t0)
