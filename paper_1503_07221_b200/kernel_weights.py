"""psi / psi~ prototype tables (piecewise Chebyshev, degree 16) and light-cone supports.

Host-side, once per (dt, p): the tables are the only time-dependent input of the
assembly kernel.  The device kernel evaluates them with the Clenshaw recurrence.

Reference interface (``tdbem.kernel_weights``,
/root/reference/pkg/src/tdbem/kernel_weights.py):
  clenshaw                 :51-65
  _lobatto_matrix          :68-78   Chebyshev-Lobatto values -> coefficients
  PiecewiseCheb            :81-123
  table_domain             :163-185
  PrototypeTables          :188-322 (build :243-295, resolve :297-312)
  tables_for               :330-339 (cache keyed by (dt, p))
  is_zero_pair             :351-354
  psi_support              :381-385

The build restates the reference's quadrature exactly (32-point Gauss panels,
panel ends affine in the offset, split at dt multiples, ceil(4*len/dt)
sub-panels) so the coefficients agree to rounding (pinned against the
reference's own tables in tests/golden/tables_*.npz).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .temporal_basis import (
    KIND_FIRST,
    KIND_INNER,
    KIND_LAST,
    TimeGrid,
    canonical_basis_all,
    canonical_support,
)

__all__ = [
    "KINDS",
    "PiecewiseCheb",
    "PrototypeTables",
    "build_tables",
    "tables_for",
    "table_domain",
    "clenshaw",
    "is_zero_pair",
    "psi_support",
]

KINDS = (KIND_FIRST, KIND_INNER, KIND_LAST)


def clenshaw(coeffs, x):
    """sum_k c_k T_k(x) by the backward recurrence; x clamped into [-1, 1]."""
    x = np.asarray(x, dtype=float)
    if np.any(np.abs(x) > 1.0 + 1e-12):
        raise ValueError("Clenshaw argument outside [-1, 1]")
    x = np.clip(x, -1.0, 1.0)
    b1 = np.zeros_like(x)
    b2 = np.zeros_like(x)
    for c in coeffs[:0:-1]:
        b1, b2 = 2.0 * x * b1 - b2 + c, b1
    return x * b1 - b2 + coeffs[0]


@lru_cache(maxsize=None)
def lobatto_transform(deg: int) -> tuple[np.ndarray, np.ndarray]:
    """Nodes cos(pi j/deg) and the DCT-I matrix mapping node values to coefficients."""
    j = np.arange(deg + 1)
    nodes = np.cos(np.pi * j / deg)
    D = (2.0 / deg) * np.cos(np.pi * np.outer(j, j) / deg)
    D[:, [0, deg]] *= 0.5
    D[[0, deg], :] *= 0.5
    return nodes, D


@dataclass(frozen=True)
class PiecewiseCheb:
    """Chebyshev expansions on n_sub equal subintervals of [lo, hi]."""

    lo: float
    hi: float
    coeffs: np.ndarray  # (n_sub, deg+1)

    @property
    def n_sub(self) -> int:
        return self.coeffs.shape[0]

    @property
    def width(self) -> float:
        return (self.hi - self.lo) / self.n_sub

    def __call__(self, a):
        a = np.asarray(a, dtype=float)
        scalar = a.ndim == 0
        a = np.atleast_1d(a)
        out = np.zeros_like(a)
        m = (a >= self.lo) & (a <= self.hi)
        if np.any(m):
            am = a[m]
            w = self.width
            idx = np.minimum(((am - self.lo) / w).astype(np.int64), self.n_sub - 1)
            x = np.clip(2.0 * (am - self.lo - idx * w) / w - 1.0, -1.0, 1.0)
            c = self.coeffs[idx]  # (n, deg+1)
            b1 = np.zeros_like(x)
            b2 = np.zeros_like(x)
            for k in range(c.shape[1] - 1, 0, -1):
                b1, b2 = 2.0 * x * b1 - b2 + c[:, k], b1
            out[m] = x * b1 - b2 + c[:, 0]
        return float(out[0]) if scalar else out


def table_domain(grid: TimeGrid, kind_i: str, kind_k: str):
    """Stored offset range of a (ansatz kind, test kind) prototype, or None.

    Natural support [-len_i, len_k]; inner/inner keeps the folded half
    [0, 2dt]; last-ansatz variants start at dt (inner test) or 0 (last test);
    a first-kind test starts at 0; last/first is unreachable.
    """
    len_i = canonical_support(grid, kind_i)
    len_k = canonical_support(grid, kind_k)
    if kind_i == KIND_INNER and kind_k == KIND_INNER:
        return 0.0, len_k
    if kind_i == KIND_LAST:
        if kind_k == KIND_FIRST:
            return None
        return (grid.dt if kind_k == KIND_INNER else 0.0), len_k
    if kind_k == KIND_FIRST:
        return 0.0, len_k
    return -len_i, len_k


class PrototypeTables:
    """All prototype tables of one grid, keyed (tilde, kind_i, kind_k, m1, m2).

    tilde=False: int b_i''(u - a) b_k'(u) du  (psi, pairs with n_x.n_y)
    tilde=True : int b_i(u - a)   b_k'(u) du  (psi~, pairs with the curls)
    m1 = ansatz order (kind_i), m2 = test order (kind_k).
    """

    def __init__(self, grid: TimeGrid, deg: int = 16, n_per_step: int = 8,
                 n_per_step_boundary: int = 32, nq: int = 32):
        self.grid = grid
        self.deg = deg
        self.n_per_step = n_per_step
        self.n_per_step_boundary = n_per_step_boundary
        self.nq = nq
        self.tables: dict = {}

    def key_iter(self):
        p = self.grid.p
        for tilde in (True, False):
            for ki in KINDS:
                for kk in KINDS:
                    for m1 in range(p + 1):
                        for m2 in range(p + 1):
                            if ki == KIND_INNER and kk == KIND_INNER and m1 > m2:
                                continue
                            yield tilde, ki, kk, m1, m2

    # -- quadrature of the defining integral ---------------------------------
    def _panels(self, kind_i: str, kind_k: str, a_mid: float):
        """Breakpoints of u in [max(0,a), min(len_k, a+len_i)] as affine (c, s): c + s*a.

        The ordering of the breakpoints is fixed inside one table subinterval
        (crossings happen only at dt multiples, which are subinterval edges),
        so it is decided at the subinterval midpoint a_mid.
        """
        dt = self.grid.dt
        len_i = canonical_support(self.grid, kind_i)
        len_k = canonical_support(self.grid, kind_k)
        lo = (0.0, 1.0) if a_mid > 0.0 else (0.0, 0.0)
        hi = (len_i, 1.0) if a_mid + len_i < len_k else (len_k, 0.0)

        def at(e):
            return e[0] + e[1] * a_mid

        cand = [(j * dt, 0.0) for j in range(int(round(len_k / dt)) + 1)]
        cand += [(j * dt, 1.0) for j in range(int(round(len_i / dt)) + 1)]
        mids = sorted((e for e in cand if at(lo) < at(e) < at(hi)), key=at)
        ends = [lo] + mids + [hi]
        return [(ends[k], ends[k + 1]) for k in range(len(ends) - 1)], at

    def _node_values(self, kind_i, kind_k, a0, width, nodes, xq, wq):
        """Both prototype variants at the Lobatto nodes of one subinterval.

        Returns (2, p+1, p+1, deg+1): [variant(psi, psi~), m1, m2, node].
        """
        p = self.grid.p
        dt = self.grid.dt
        alpha = a0 + 0.5 * width * (nodes + 1.0)
        a_mid = a0 + 0.5 * width
        out = np.zeros((2, p + 1, p + 1, len(nodes)))
        panels, at = self._panels(kind_i, kind_k, a_mid)
        for e0, e1 in panels:
            ua = e0[0] + e0[1] * alpha
            ub = e1[0] + e1[1] * alpha
            n_split = max(1, math.ceil(4.0 * (at(e1) - at(e0)) / dt))
            for j in range(n_split):
                qa = ua + (ub - ua) * (j / n_split)
                qb = ua + (ub - ua) * ((j + 1) / n_split)
                h = 0.5 * (qb - qa)
                U = 0.5 * (qa + qb)[:, None] + h[:, None] * xq[None, :]
                W = np.maximum(h, 0.0)[:, None] * wq[None, :]
                S = U - alpha[:, None]
                test = W[None] * canonical_basis_all(self.grid, kind_k, p, U, 1)
                d2 = canonical_basis_all(self.grid, kind_i, p, S, 2)
                d0 = canonical_basis_all(self.grid, kind_i, p, S, 0)
                out[0] += np.einsum("inq,knq->ikn", d2, test)
                out[1] += np.einsum("inq,knq->ikn", d0, test)
        return out

    def build_device(self, ctx=None) -> "PrototypeTables":
        """Same tables with the node integrals evaluated on the GPU (csrc/tdb_tables.cu):
        the panel structure is decided here per subinterval exactly as in build();
        the values agree with the host build to rounding (~1e-15 of the table max)."""
        from . import _lib

        grid = self.grid
        p = grid.p
        dt = grid.dt
        nodes, D = lobatto_transform(self.deg)
        xq, wq = np.polynomial.legendre.leggauss(self.nq)
        kind_id = {k: i for i, k in enumerate(KINDS)}
        kinds, a0w, pptr, panels, fams = [], [], [0], [], []
        for kind_i in KINDS:
            for kind_k in KINDS:
                dom = table_domain(grid, kind_i, kind_k)
                if dom is None or dom[1] <= dom[0]:
                    for tilde in (True, False):
                        for m1 in range(p + 1):
                            for m2 in range(p + 1):
                                self.tables[(tilde, kind_i, kind_k, m1, m2)] = None
                    continue
                lo, hi = dom
                boundary = not (kind_i == KIND_INNER and kind_k == KIND_INNER)
                per = self.n_per_step_boundary if boundary else self.n_per_step
                n_sub = max(1, round((hi - lo) / grid.dt * per))
                width = (hi - lo) / n_sub
                fams.append((kind_i, kind_k, lo, hi, n_sub, len(kinds)))
                for ks in range(n_sub):
                    a0 = lo + ks * width
                    a_mid = a0 + 0.5 * width
                    pl, at = self._panels(kind_i, kind_k, a_mid)
                    for e0, e1 in pl:
                        panels.append((e0[0], e0[1], e1[0], e1[1],
                                       float(max(1, math.ceil(4.0 * (at(e1) - at(e0)) / dt)))))
                    kinds.append((kind_id[kind_i], kind_id[kind_k]))
                    a0w.append((a0, width))
                    pptr.append(len(panels))
        nsub = len(kinds)
        out = np.empty((nsub, 2, p + 1, p + 1, len(nodes)))
        ctx = ctx or _lib.default_context()
        arr = dict(kinds=np.ascontiguousarray(kinds, dtype=np.int32), a0w=_lib.f64(a0w), nodes=_lib.f64(nodes),
                   pptr=np.ascontiguousarray(pptr, dtype=np.int32), panels=_lib.f64(panels), xq=_lib.f64(xq),
                   wq=_lib.f64(wq))
        _lib.check(_lib.LIB.tdb_table_node_values(
            ctx.handle, float(dt), int(p), int(nsub), _lib.ptr(arr["kinds"], _lib.C.c_int32), _lib.ptr(arr["a0w"]),
            len(nodes), _lib.ptr(arr["nodes"]), _lib.ptr(arr["pptr"], _lib.C.c_int32), _lib.ptr(arr["panels"]),
            len(xq), _lib.ptr(arr["xq"]), _lib.ptr(arr["wq"]), _lib.ptr(out)), "table_node_values")
        for kind_i, kind_k, lo, hi, n_sub, s0 in fams:
            vals = np.moveaxis(out[s0 : s0 + n_sub], 0, 3)  # (2, p+1, p+1, n_sub, nodes)
            coeffs = np.einsum("ij,vabkj->vabki", D, vals)
            pairs = [(m1, m2) for m1 in range(p + 1) for m2 in range(p + 1)
                     if not (kind_i == KIND_INNER and kind_k == KIND_INNER and m1 > m2)]
            for m1, m2 in pairs:
                self.tables[(False, kind_i, kind_k, m1, m2)] = PiecewiseCheb(lo, hi, coeffs[0, m1, m2])
                self.tables[(True, kind_i, kind_k, m1, m2)] = PiecewiseCheb(lo, hi, coeffs[1, m1, m2])
        return self

    def build(self) -> "PrototypeTables":
        grid = self.grid
        p = grid.p
        nodes, D = lobatto_transform(self.deg)
        xq, wq = np.polynomial.legendre.leggauss(self.nq)
        for kind_i in KINDS:
            for kind_k in KINDS:
                dom = table_domain(grid, kind_i, kind_k)
                pairs = [(m1, m2) for m1 in range(p + 1) for m2 in range(p + 1)
                         if not (kind_i == KIND_INNER and kind_k == KIND_INNER and m1 > m2)]
                if dom is None or dom[1] <= dom[0]:
                    for tilde in (True, False):
                        for m1 in range(p + 1):
                            for m2 in range(p + 1):
                                self.tables[(tilde, kind_i, kind_k, m1, m2)] = None
                    continue
                lo, hi = dom
                boundary = not (kind_i == KIND_INNER and kind_k == KIND_INNER)
                per = self.n_per_step_boundary if boundary else self.n_per_step
                n_sub = max(1, round((hi - lo) / grid.dt * per))
                width = (hi - lo) / n_sub
                vals = np.zeros((2, p + 1, p + 1, n_sub, self.deg + 1))
                for ks in range(n_sub):
                    vals[:, :, :, ks, :] = self._node_values(
                        kind_i, kind_k, lo + ks * width, width, nodes, xq, wq)
                coeffs = np.einsum("ij,vabkj->vabki", D, vals)
                for m1, m2 in pairs:
                    self.tables[(False, kind_i, kind_k, m1, m2)] = PiecewiseCheb(lo, hi, coeffs[0, m1, m2])
                    self.tables[(True, kind_i, kind_k, m1, m2)] = PiecewiseCheb(lo, hi, coeffs[1, m1, m2])
        return self

    def resolve(self, tilde: bool, kind_i: str, kind_k: str, m1: int, m2: int):
        """(table, sign for a >= 0, sign for a < 0, fold) of one weight evaluation.

        Inner/inner stores m1 <= m2 on a >= 0 only; the order-swap and parity
        symmetries psi_{m1,m2}(-a) = -psi_{m2,m1}(a) = (-1)^(m1+m2+1) psi_{m1,m2}(a)
        give the rest (kernel_weights.py:297-312).
        """
        if kind_i == KIND_INNER and kind_k == KIND_INNER:
            par = -1.0 if (m1 + m2) % 2 else 1.0
            if m1 <= m2:
                return self.tables[(tilde, kind_i, kind_k, m1, m2)], 1.0, -par, True
            return self.tables[(tilde, kind_i, kind_k, m2, m1)], par, -1.0, True
        return self.tables[(tilde, kind_i, kind_k, m1, m2)], 1.0, 1.0, False

    def eval_offset(self, tilde, kind_i, kind_k, m1, m2, a):
        tbl, sp, sn, fold = self.resolve(tilde, kind_i, kind_k, m1, m2)
        a = np.asarray(a, dtype=float)
        if tbl is None:
            return np.zeros_like(a) if a.ndim else 0.0
        if not fold:
            return tbl(a)
        return np.where(a >= 0.0, sp * tbl(a), sn * tbl(-a))


def build_tables(grid: TimeGrid, **kwargs) -> PrototypeTables:
    return PrototypeTables(grid, **kwargs).build()


_CACHE: dict = {}


def _device_ok() -> bool:
    try:
        import torch

        return bool(torch.cuda.is_available())
    except ImportError:
        return False


def tables_for(grid: TimeGrid, device: bool | None = None) -> PrototypeTables:
    """Default-parameter tables, cached by (dt, p) (independent of N).

    device=None: built on the GPU when one is visible (build_device), else on the
    host (build: bit-identical to the reference's tables)."""
    use_dev = _device_ok() if device is None else bool(device)
    key = (round(grid.dt, 15), grid.p, use_dev)
    if key not in _CACHE:
        _CACHE[key] = PrototypeTables(grid).build_device() if use_dev else build_tables(grid)
    return _CACHE[key]


def is_zero_pair(grid: TimeGrid, k_tilde: int, i_tilde: int) -> bool:
    """Causality: the test support ends no later than the ansatz support starts."""
    return grid.t_formal(k_tilde) <= grid.t_formal(i_tilde - 2)


def psi_support(grid: TimeGrid, k_tilde: int, i_tilde: int) -> tuple[float, float]:
    """Distance support [max(0, t_{k-2} - t_i), t_k - t_{i-2}] of the block weights."""
    lo = max(0.0, grid.t_formal(k_tilde - 2) - grid.t_formal(i_tilde))
    return lo, grid.t_formal(k_tilde) - grid.t_formal(i_tilde - 2)
