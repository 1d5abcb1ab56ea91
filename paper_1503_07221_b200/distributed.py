"""Sharding over GPUs by row blocks and lags: one process per GPU, NCCL over NVLink.

Assembly needs no communication: rank r owns a set of test-vertex rows J_r and
assembles exactly those CSR rows of every canonical block from the pairs whose
test triangle lies in a star of J_r (tdb_system_create with `rows`).  Rows are
owned by the lowest-numbered adjacent triangle, and triangles are split into
contiguous blocks; refinement numbers children of one parent consecutively, so
blocks are spatially compact and the halo (test triangles shared between
ranks, computed twice) stays small.

Vectors are distributed the same way: each rank holds x[time][J_r].  A matvec
all-gathers the iterate (one ncclAllGather of L*(p+1)*max|J_r| doubles into a
rank-major buffer), the kernel reads it through an index map (no reshuffle
copy) and produces the rank's rows of y.  Krylov dots/norms are all-reduced
(solvers.TorchDistComm).

Lag split (the north star's "by lag and row blocks"; the paper's diagonal-wise block
ownership, PAPER.md 5.1 / ref/block_system.py:86-129): with lag_groups = G the world
is R x G, rank = rb * G + lg.  Rank (rb, lg) assembles the rows of row block rb for
the lg-th contiguous lag range of every table family only (partition_lags).  Its
matvec produces the partial rows over those lags, summed over the G ranks of the row
block by one all-reduce (the paper's gather-sum); the iterate is
all-gathered within the row group (the R ranks sharing lg), and Krylov dot products
are all-reduced over the row group too (vectors are replicated over the lag group).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .assembly import DeviceAssembly, QuadratureConfig, as_product_inputs, build_plan
from .block_system import canonical_position, canonical_positions, is_zero_position
from .kernel_weights import tables_for

__all__ = ["partition_rows", "partition_lags", "gathered_x_map", "make_groups", "DistributedBlockHessenbergMatrix",
           "assemble_system_distributed"]


def partition_rows(mesh, nparts: int):
    """Owned vertex rows per rank (sorted) and their test triangles (sorted)."""
    E, V = mesh.num_triangles, mesh.num_vertices
    tri = np.asarray(mesh.triangles)
    owner_tri = np.full(V, E, dtype=np.int64)
    for a in range(3):
        np.minimum.at(owner_tri, tri[:, a], np.arange(E))
    # vertices in owner-triangle order (refinement numbers a parent's children
    # consecutively, so runs of this order are spatially compact), cut into equal
    # counts: every rank owns V / nparts rows (+-1)
    order = np.argsort(owner_tri, kind="stable")
    cuts = [(V * r) // nparts for r in range(nparts + 1)]
    rows = [np.sort(order[cuts[r]:cuts[r + 1]]).astype(np.int64) for r in range(nparts)]
    off, ids = mesh.star_csr
    tests = []
    for r in range(nparts):
        need = np.zeros(E, dtype=bool)
        for j in rows[r]:
            need[ids[off[j] : off[j + 1]]] = True
        tests.append(np.flatnonzero(need))
    return rows, tests


def partition_lags(grid, positions, groups: int):
    """Canonical positions -> `groups` lists: every table family (positions sharing
    (ansatz kind, test kind), in lag order) cut into contiguous lag ranges of near-equal
    length, so each group keeps consecutive lags (the band tiles need them) and the
    small-lag positions carrying the singular pairs are spread over the ranges of every
    family."""
    from .temporal_basis import timestep_kind

    fams: dict = {}
    for kt, it in positions:
        fams.setdefault((timestep_kind(grid, it), timestep_kind(grid, kt)), []).append((kt, it))
    out = [[] for _ in range(groups)]
    for key in sorted(fams):
        pos = sorted(fams[key], key=lambda p: p[0] - p[1])
        n = len(pos)
        for g in range(groups):
            out[g] += pos[(n * g) // groups:(n * (g + 1)) // groups]
    return [sorted(o) for o in out]


def make_groups(rows: int, lags: int):
    """torch.distributed process groups of a rows x lags world (every rank calls this):
    (row group of this rank: the `rows` ranks sharing its lag group, lag group of this
    rank: the `lags` ranks sharing its row block)."""
    import torch.distributed as dist

    rank = dist.get_rank()
    mine_row = mine_lag = None
    for lg in range(lags):
        g = dist.new_group([rb * lags + lg for rb in range(rows)])
        if rank % lags == lg:
            mine_row = g
    for rb in range(rows):
        g = dist.new_group([rb * lags + lg for lg in range(lags)])
        if rank // lags == rb:
            mine_lag = g
    return mine_row, mine_lag


def gathered_x_map(rows_per_rank, M: int, ncols: int, nmax: int) -> np.ndarray:
    """x_map for the all-gathered rank-major layout [rank][column][nmax] (TdbMatvecDesc)."""
    xmap = np.empty(M, dtype=np.int64)
    for r, rows in enumerate(rows_per_rank):
        xmap[rows] = r * ncols * nmax + np.arange(len(rows))
    return xmap


class _DistMatvecPlan:
    def __init__(self, A: "DistributedBlockHessenbergMatrix", rows, cols):
        grid = A.grid
        rlo, rhi = rows
        clo, chi = cols
        words = (grid.N + 31) // 32
        where = A.dev.plan.where
        terms: dict = {}
        for kt in range(rlo, rhi + 1):
            for it in range(max(clo, kt - grid.N), min(chi, kt + 1) + 1):
                if is_zero_position(grid, A.diameter, kt, it):
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
        self.handle = None
        self.bytes = 0.0
        self.flops = 0.0
        self.ncols = (chi - clo + 1) * (grid.p + 1)
        if not keys:
            return
        tf = np.array([k[0] for k in keys], dtype=np.int32)
        ts = np.array([k[1] for k in keys], dtype=np.int32)
        td = np.array([k[2] for k in keys], dtype=np.int32)
        tm = np.ascontiguousarray(np.stack([terms[k] for k in keys]))
        self.xmap = gathered_x_map(A.rows_per_rank, A.M_global, self.ncols, A.nmax)
        desc = _lib.TdbMatvecDesc()
        desc.N, desc.rlo, desc.rhi, desc.clo, desc.chi = grid.N, rlo, rhi, clo, chi
        desc.nterms, desc.words = len(keys), words
        desc.term_family, desc.term_pos = _lib.ptr(tf, C.c_int32), _lib.ptr(ts, C.c_int32)
        desc.term_d, desc.term_mask = _lib.ptr(td, C.c_int32), _lib.ptr(tm, C.c_uint32)
        desc.x_stride = A.nmax
        desc.x_map = _lib.ptr(self.xmap, C.c_int64)
        h = C.c_void_p()
        _lib.check(_lib.LIB.tdb_matvec_plan_create(A.dev.handle, C.byref(desc), C.byref(h)), "matvec_plan_create")
        self.handle = h
        b, f = C.c_double(), C.c_double()
        _lib.check(_lib.LIB.tdb_matvec_plan_work(h, C.byref(b), C.byref(f)), "matvec_plan_work")
        self.bytes, self.flops = b.value, f.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib.LIB is not None:  # LIB is None at interpreter exit
            _lib.LIB.tdb_matvec_plan_destroy(h)
            self.handle = None


class DistributedBlockHessenbergMatrix:
    """This rank's share of the block Hessenberg matrix (duck-types BlockHessenbergMatrix
    for the solvers: .grid, .M (local rows), .matvec(x_local, rows, cols)).

    rows_per_rank: the R row blocks (partition_rows); rank = rb * lag_groups + lg.
    row_group / lag_group: torch.distributed groups (make_groups) for the all-gather of
    the iterate and the partial-row sum; gather / reduce callbacks replace them (tests).
    """

    def __init__(self, mesh, grid, rows_per_rank, rank: int, ctx=None, tables=None,
                 config: QuadratureConfig = QuadratureConfig(), gather=None, lag_groups: int = 1,
                 row_group=None, lag_group=None, reduce=None, create_only: bool = False):
        mesh, grid = as_product_inputs(mesh, grid)
        self.grid = grid
        self.diameter = mesh.diameter
        self.rank = rank
        self.lag_groups = lag_groups
        self.rb, self.lg = rank // lag_groups, rank % lag_groups
        self.rows_per_rank = rows_per_rank
        self.nparts = len(rows_per_rank)
        self.rows = rows_per_rank[self.rb]
        self.M_global = mesh.num_vertices
        self.M = len(self.rows)  # local rows (what the solvers' half-splits use)
        self.nmax = max(len(r) for r in rows_per_rank)
        tables = tables_for(grid) if tables is None else tables
        positions = canonical_positions(grid, mesh.diameter)
        if lag_groups > 1:
            positions = partition_lags(grid, positions, lag_groups)[self.lg]
        plan = build_plan(mesh, grid, tables, positions, config)
        self.dev = DeviceAssembly(mesh, plan, ctx or _lib.default_context(), rows=self.rows, create_only=create_only)
        self._plans: dict = {}
        # gather(local_padded (ncols, nmax) tensor) -> (nparts, ncols, nmax) tensor
        self._gather = gather
        self._reduce = reduce
        self.row_group, self.lag_group = row_group, lag_group

    @property
    def shape_local(self):
        return (self.grid.L * self.M, self.grid.L * self.M_global)

    def _plan(self, rows, cols):
        key = (tuple(rows), tuple(cols))
        p = self._plans.get(key)
        if p is None:
            p = self._plans[key] = _DistMatvecPlan(self, rows, cols)
        return p

    def allgather(self, x_local: torch.Tensor, ncols: int) -> torch.Tensor:
        pad = torch.zeros((ncols, self.nmax), dtype=x_local.dtype, device=x_local.device)
        pad[:, : self.M] = x_local.view(ncols, self.M)
        if self._gather is not None:
            return self._gather(pad)
        import torch.distributed as dist

        if dist.get_backend(self.row_group) != "nccl":  # gloo: host-staged (tests / plumbing checks)
            parts = [torch.empty_like(pad, device="cpu") for _ in range(self.nparts)]
            dist.all_gather(parts, pad.cpu(), group=self.row_group)
            return torch.stack(parts).to(x_local.device)
        out = torch.empty((self.nparts, ncols, self.nmax), dtype=x_local.dtype, device=x_local.device)
        dist.all_gather_into_tensor(out, pad.contiguous(), group=self.row_group)
        return out

    def reduce_lags(self, y: torch.Tensor) -> torch.Tensor:
        """Sum the partial rows over the lag group (the paper's gather-sum)."""
        if self.lag_groups == 1:
            return y
        if self._reduce is not None:
            return self._reduce(y)
        import torch.distributed as dist

        if dist.get_backend(self.lag_group) != "nccl":  # gloo: host-staged
            c = y.cpu()
            dist.all_reduce(c, group=self.lag_group)
            y.copy_(c)
            return y
        dist.all_reduce(y, group=self.lag_group)
        return y

    def matvec(self, x_local: torch.Tensor, rows=None, cols=None) -> torch.Tensor:
        np1 = self.grid.p + 1
        rlo, rhi = rows if rows is not None else (1, self.grid.N)
        clo, chi = cols if cols is not None else (1, self.grid.N)
        ncols = (chi - clo + 1) * np1
        if x_local.numel() != ncols * self.M:
            raise ValueError("matvec dimension mismatch")
        plan = self._plan((rlo, rhi), (clo, chi))
        xg = self.allgather(x_local.contiguous(), ncols).contiguous()
        nrow = (rhi - rlo + 1) * np1 * self.M
        y = torch.zeros(nrow, dtype=x_local.dtype, device=x_local.device)
        if plan.handle is not None and nrow:
            self.dev.ctx.set_stream(torch.cuda.current_stream(x_local.device).cuda_stream)
            _lib.check(_lib.LIB.tdb_matvec(plan.handle, C.c_void_p(xg.data_ptr()), C.c_void_p(y.data_ptr())),
                       "matvec")
        return self.reduce_lags(y)

    def __matmul__(self, x):
        return self.matvec(x)

    def local_of(self, x_full: np.ndarray, ncols: int | None = None) -> np.ndarray:
        """This rank's piece [column][J_r] of a time-major global vector."""
        ncols = ncols or self.grid.L
        return np.ascontiguousarray(np.asarray(x_full).reshape(ncols, self.M_global)[:, self.rows]).ravel()

    def stats(self) -> dict:
        return self.dev.stats()


def assemble_system_distributed(mesh, grid, rank: int, world: int, ctx=None, tables=None,
                                config: QuadratureConfig = QuadratureConfig(), lag_groups: int = 1,
                                create_only: bool = False):
    """Assemble this rank's (row block, lag range) share; torch.distributed must be
    initialised (every rank calls this: it creates the process groups)."""
    mesh, grid = as_product_inputs(mesh, grid)
    if world % lag_groups:
        raise ValueError(f"lag_groups {lag_groups} must divide the world size {world}")
    rows, _ = partition_rows(mesh, world // lag_groups)
    row_group = lag_group = None
    if lag_groups > 1:
        row_group, lag_group = make_groups(world // lag_groups, lag_groups)
    return DistributedBlockHessenbergMatrix(mesh, grid, rows, rank, ctx=ctx, tables=tables, config=config,
                                            lag_groups=lag_groups, row_group=row_group, lag_group=lag_group,
                                            create_only=create_only)
