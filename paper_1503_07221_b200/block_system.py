"""Block Hessenberg system: canonical lag blocks on the device + device matvec.

Reference interface (``tdbem.block_system``,
/root/reference/pkg/src/tdbem/block_system.py):
  n_tilde_z / inner_nonzero_count   :37-47
  canonical_position                :54-66
  DistributionPlan/plan_distribution:69-129
  BlockHessenbergMatrix             :132-219 (is_zero_position :153-160,
                                              resolve :162-172, matvec :180-216)
  assemble_system                   :228-275
  reconstruct_dense                 :278-296

The canonical blocks live in device memory (libtdb TdbSystem, CSR per table
family); ``matvec`` runs csrc/tdb_matvec.cu on device vectors (torch CUDA
tensors) and accepts/returns numpy arrays for reference-style callers.
``unique_blocks`` materialises the reference's nested scipy CSR lists lazily
(inner canonical positions keep m1 <= m2 only, as the reference does).
"""

from __future__ import annotations

import ctypes as C
import functools
import os
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib
from .assembly import DeviceAssembly, QuadratureConfig, build_plan
from .kernel_weights import PrototypeTables, is_zero_pair, tables_for
from .mesh import SurfaceMesh
from .temporal_basis import TimeGrid

__all__ = [
    "BlockHessenbergMatrix",
    "DistributionPlan",
    "plan_distribution",
    "assemble_system",
    "reconstruct_dense",
    "canonical_position",
    "canonical_positions",
    "n_tilde_z",
    "inner_nonzero_count",
]


def n_tilde_z(grid: TimeGrid, diameter: float) -> int:
    """Non-zero block count of the first matrix column."""
    return min(grid.N, int(np.ceil(2.0 * diameter / grid.dt)) + 2)


def inner_nonzero_count(n: int, ntz: int) -> int:
    """Closed-form count of inner positions 2 <= it, kt <= N-1 with -1 <= kt-it < ntz."""
    return (n * n - n - 4) // 2 - ((n - ntz - 2) * max(n - ntz - 1, 0)) // 2


def _inner(grid: TimeGrid, t: int) -> bool:
    return 1 < t < grid.N


def canonical_position(grid: TimeGrid, kt: int, it: int):
    """Stored position for logical (kt, it): inner blocks reuse (kt-it+2, 2) or (2, 3)."""
    if kt - it <= -2:
        return None
    if _inner(grid, kt) and _inner(grid, it):
        return (kt - it + 2, 2) if kt >= it else (2, 3)
    return (kt, it)


def is_zero_position(grid: TimeGrid, diameter: float, kt: int, it: int) -> bool:
    """Hessenberg band + causality + light-cone cut, with the reference's FP64 expressions."""
    if kt - it <= -2:
        return True
    if is_zero_pair(grid, kt, it):
        return True
    return grid.t_formal(kt - 2) - grid.t_formal(it) > diameter


def canonical_positions(grid: TimeGrid, diameter: float) -> list:
    """Sorted canonical block positions (pure function of the grid and the diameter,
    cached: repeated assemblies of one system skip the O(N^2) predicate loop)."""
    return list(_canonical_positions(grid, float(diameter)))


@functools.lru_cache(maxsize=64)
def _canonical_positions(grid: TimeGrid, diameter: float) -> tuple:
    pos = set()
    for kt in range(1, grid.N + 1):
        for it in range(max(1, kt - grid.N), min(grid.N, kt + 1) + 1):
            if is_zero_position(grid, diameter, kt, it):
                continue
            c = canonical_position(grid, kt, it)
            if c is not None:
                pos.add(c)
    return tuple(sorted(pos))


@dataclass(frozen=True)
class DistributionPlan:
    """Diagonal-wise ownership of block positions across P ranks (paper 5.1)."""

    P: int
    n_z: int
    n_tilde_z: int
    owners: dict

    def rank_loads(self, grid: TimeGrid) -> np.ndarray:
        loads = np.zeros(self.P, dtype=np.int64)
        for (kt, it), r in self.owners.items():
            if _inner(grid, kt) and _inner(grid, it):
                loads[r] += 1
        return loads


def plan_distribution(grid: TimeGrid, mesh: SurfaceMesh, P: int) -> DistributionPlan:
    """Inner positions diagonal by diagonal in P contiguous near-equal chunks;
    boundary positions greedily to the least-loaded rank (block_system.py:86-129).
    The mesh enters only through its diameter, so the plan is cached on (grid, diameter, P)."""
    if P < 1:
        raise ValueError(f"worker count {P} must be >= 1")
    return _plan_distribution(grid, float(mesh.diameter), int(P))


@functools.lru_cache(maxsize=64)
def _plan_distribution(grid: TimeGrid, diameter: float, P: int) -> DistributionPlan:
    n = grid.N
    ntz = n_tilde_z(grid, diameter)
    inner = [(it + d, it) for d in range(-1, ntz) for it in range(2, n) if 2 <= it + d <= n - 1]
    owners = {}
    base, extra = divmod(len(inner), P)
    loads = np.zeros(P, dtype=np.int64)
    k = 0
    for r in range(P):
        size = base + (1 if r < extra else 0)
        for pos in inner[k : k + size]:
            owners[pos] = r
        loads[r] = size
        k += size
    boundary = sorted(
        (kt, it)
        for kt in range(1, n + 1)
        for it in range(1, n + 1)
        if not (_inner(grid, kt) and _inner(grid, it)) and -2 < kt - it < ntz
    )
    for pos in boundary:
        r = int(np.argmin(loads))
        owners[pos] = r
        loads[r] += 1
    return DistributionPlan(P=P, n_z=len(inner), n_tilde_z=ntz, owners=owners)


class _MatvecPlan:
    """libtdb matvec plan for one (rows, cols) block range."""

    def __init__(self, A: "BlockHessenbergMatrix", rows, cols):
        grid = A.grid
        self.rows, self.cols = rows, cols
        self.tiled_terms = self.csr_terms = 0
        rlo, rhi = rows
        clo, chi = cols
        words = (grid.N + 31) // 32
        terms: dict = {}
        where = A._dev.plan.where if A._dev is not None else {}
        for kt in range(rlo, rhi + 1):
            for it in range(max(clo, kt - grid.N), min(chi, kt + 1) + 1):
                if A.is_zero_position(kt, it):
                    continue
                c = canonical_position(grid, kt, it)
                loc = where.get(c) if c is not None else None
                if loc is None:
                    continue
                key = (loc[0], loc[1], kt - it)
                m = terms.get(key)
                if m is None:
                    m = terms[key] = np.zeros(words, dtype=np.uint32)
                m[(kt - 1) // 32] |= np.uint32(1 << ((kt - 1) % 32))
        keys = sorted(terms)
        self.nterms = len(keys)
        self.handle = None
        self.bytes = 0.0
        self.flops = 0.0
        if not keys:
            return
        tf = np.array([k[0] for k in keys], dtype=np.int32)
        ts = np.array([k[1] for k in keys], dtype=np.int32)
        td = np.array([k[2] for k in keys], dtype=np.int32)
        tm = np.ascontiguousarray(np.stack([terms[k] for k in keys]))
        desc = _lib.TdbMatvecDesc()
        desc.N, desc.rlo, desc.rhi, desc.clo, desc.chi = grid.N, rlo, rhi, clo, chi
        desc.nterms, desc.words = len(keys), words
        desc.term_family = _lib.ptr(tf, C.c_int32)
        desc.term_pos = _lib.ptr(ts, C.c_int32)
        desc.term_d = _lib.ptr(td, C.c_int32)
        desc.term_mask = _lib.ptr(tm, C.c_uint32)
        h = C.c_void_p()
        _lib.check(_lib.LIB.tdb_matvec_plan_create(A._dev.handle, C.byref(desc), C.byref(h)),
                   "matvec_plan_create")
        self.handle = h
        b, f = C.c_double(), C.c_double()
        _lib.check(_lib.LIB.tdb_matvec_plan_work(h, C.byref(b), C.byref(f)), "matvec_plan_work")
        self.bytes, self.flops = b.value, f.value
        nt_, nc_ = C.c_int32(0), C.c_int32(0)
        _lib.check(_lib.LIB.tdb_matvec_plan_kind(h, C.byref(nt_), C.byref(nc_)), "matvec_plan_kind")
        self.tiled_terms, self.csr_terms = nt_.value, nc_.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib.LIB is not None:  # LIB is None at interpreter exit
            _lib.LIB.tdb_matvec_plan_destroy(h)
            self.handle = None


@dataclass
class BlockHessenbergMatrix:
    """Global matrix as device-resident canonical blocks plus reuse metadata."""

    grid: TimeGrid
    M: int
    diameter: float
    plan: DistributionPlan | None = None
    _dev: DeviceAssembly | None = None
    _unique: dict | None = field(default=None, repr=False)
    _mv_plans: dict = field(default_factory=dict, repr=False)

    @property
    def shape(self) -> tuple[int, int]:
        n = self.grid.L * self.M
        return (n, n)

    def is_zero_position(self, kt: int, it: int) -> bool:
        return is_zero_position(self.grid, self.diameter, kt, it)

    @property
    def unique_blocks(self) -> dict:
        """(kt, it) -> (p+1) x (p+1) nested scipy CSR lists (host copies, built once)."""
        if self._unique is None:
            out = {}
            cache: dict = {}
            np1 = self.grid.p + 1
            if self._dev is not None:
                for pos in sorted(self._dev.plan.where):
                    blocks = self._dev.position_blocks(*pos, _cache=cache)
                    if _inner(self.grid, pos[0]) and _inner(self.grid, pos[1]):
                        for m2 in range(np1):
                            for m1 in range(m2 + 1, np1):
                                blocks[m2][m1] = None
                    out[pos] = blocks
            self._unique = out
        return self._unique

    def resolve(self, kt: int, it: int, m2: int, m1: int):
        pos = canonical_position(self.grid, kt, it)
        if pos is None or self.is_zero_position(kt, it):
            return None, 1.0
        stored = self.unique_blocks.get(pos)
        if stored is None:
            return None, 1.0
        if _inner(self.grid, kt) and _inner(self.grid, it) and m1 > m2:
            return stored[m1][m2], float((-1) ** (m1 + m2))
        return stored[m2][m1], 1.0

    def sub_block(self, kt: int, it: int, m2: int, m1: int) -> sp.csr_matrix:
        blk, sign = self.resolve(kt, it, m2, m1)
        if blk is None:
            return sp.csr_matrix((self.M, self.M))
        return sign * blk

    def matvec_plan(self, rows=None, cols=None) -> _MatvecPlan:
        rows = tuple(rows) if rows is not None else (1, self.grid.N)
        cols = tuple(cols) if cols is not None else (1, self.grid.N)
        key = (rows, cols)
        p = self._mv_plans.get(key)
        if p is None:
            p = self._mv_plans[key] = _MatvecPlan(self, rows, cols)
        return p

    # block rows per matvec plan (the CSR kernel's lanes cover at most 12 x 32 block rows)
    MAX_PLAN_ROWS = 384

    def matvec(self, x, rows=None, cols=None):
        """y = A[rows, cols] x; rows/cols are inclusive 1-based block ranges.

        x may be a numpy array (returns numpy) or a float64 CUDA torch tensor
        (returns a CUDA tensor, stream-ordered on torch's current stream).
        Row ranges longer than MAX_PLAN_ROWS are applied in row chunks, one plan each.
        """
        import torch

        np1 = self.grid.p + 1
        rlo, rhi = rows if rows is not None else (1, self.grid.N)
        clo, chi = cols if cols is not None else (1, self.grid.N)
        nrow = (rhi - rlo + 1) * np1 * self.M
        ncol = (chi - clo + 1) * np1 * self.M
        is_np = not isinstance(x, torch.Tensor)
        if len(x) != ncol:
            raise ValueError("matvec dimension mismatch")
        dev = torch.device("cuda", self._dev.ctx.device if self._dev else 0)
        xd = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).to(dev) if is_np else x
        if xd.dtype != torch.float64 or not xd.is_cuda or not xd.is_contiguous():
            raise ValueError("matvec expects a contiguous float64 CUDA tensor")
        y = torch.empty(nrow, dtype=torch.float64, device=xd.device)
        step = self.MAX_PLAN_ROWS
        for r0 in range(rlo, rhi + 1, step):
            r1 = min(rhi, r0 + step - 1)
            plan = self.matvec_plan((r0, r1), (clo, chi))
            ys = y[(r0 - rlo) * np1 * self.M:(r1 - rlo + 1) * np1 * self.M]
            if plan.handle is None:
                ys.zero_()
                continue
            self._dev.ctx.set_stream(torch.cuda.current_stream(xd.device).cuda_stream)
            _lib.check(_lib.LIB.tdb_matvec(plan.handle, C.c_void_p(xd.data_ptr()), C.c_void_p(ys.data_ptr())),
                       "matvec")
        return y.cpu().numpy() if is_np else y

    def __matmul__(self, x):
        return self.matvec(x)

    def stats(self) -> dict:
        return self._dev.stats() if self._dev is not None else {}


def assemble_system(mesh: SurfaceMesh, grid: TimeGrid, tables: PrototypeTables | None = None,
                    config: QuadratureConfig = QuadratureConfig(), plan: DistributionPlan | None = None,
                    workers: int | None = None, device: int | None = None) -> BlockHessenbergMatrix:
    """Assemble every canonical block position on the GPU (values independent of `workers`)."""
    from .assembly import as_product_inputs

    mesh, grid = as_product_inputs(mesh, grid)
    if workers is None:
        workers = int(os.environ.get("TDBEM_WORKERS", "1"))
    if plan is None:
        plan = plan_distribution(grid, mesh, max(1, workers))
    if tables is None:
        tables = tables_for(grid)
    positions = canonical_positions(grid, mesh.diameter)
    aplan = build_plan(mesh, grid, tables, positions, config)
    ctx = _lib.default_context(device)
    dev = DeviceAssembly(mesh, aplan, ctx)
    return BlockHessenbergMatrix(grid=grid, M=mesh.num_vertices, diameter=mesh.diameter, plan=plan, _dev=dev)


def reconstruct_dense(A: BlockHessenbergMatrix, cap: int = 20000) -> np.ndarray:
    n = A.grid.L * A.M
    if n > cap:
        raise ValueError(f"dense reconstruction of size {n} exceeds cap {cap}")
    np1 = A.grid.p + 1
    m = A.M
    out = np.zeros((n, n))
    for kt in range(1, A.grid.N + 1):
        for it in range(1, A.grid.N + 1):
            for m2 in range(np1):
                for m1 in range(np1):
                    blk, sign = A.resolve(kt, it, m2, m1)
                    if blk is None:
                        continue
                    r = ((kt - 1) * np1 + m2) * m
                    c = ((it - 1) * np1 + m1) * m
                    out[r : r + m, c : c + m] = sign * blk.toarray()
    return out
