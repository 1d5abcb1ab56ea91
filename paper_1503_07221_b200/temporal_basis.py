"""Equidistant time grid and the C-infinity temporal basis (host side).

Host-side inputs of the assembly hot path: the grid arithmetic that decides
block positions, lags and light-cone supports, and the three canonical basis
prototypes that the psi/psi~ tables are built from.

Mirrors the reference interface of ``tdbem.temporal_basis``
(/root/reference/pkg/src/tdbem/temporal_basis.py):
  TimeGrid                    temporal_basis.py:35-70
  cutoff_f                    temporal_basis.py:103-129  (erf(2 artanh t)/2 + 1/2)
  legendre_table              temporal_basis.py:132-150
  canonical_support / kind /  temporal_basis.py:202-222
  canonical_origin
  canonical_basis_all         temporal_basis.py:225-284
Only the pieces the hot path needs are here; the partition-of-unity helpers
used by the reference's RHS/postprocessing are out of scope.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
from scipy.special import erf

__all__ = [
    "TimeGrid",
    "TemporalBasisIndex",
    "flat_index",
    "decode_flat",
    "cutoff_f",
    "legendre_table",
    "timestep_kind",
    "canonical_origin",
    "canonical_support",
    "canonical_basis_all",
    "basis_b",
    "support_interval",
]

KIND_FIRST, KIND_INNER, KIND_LAST = "first", "inner", "last"

# artanh(t) is evaluated on [-1 + 1e-14, 1 - 1e-14]; at that clamp the cutoff
# has already saturated to 0/1 in double precision (temporal_basis.py:23-25).
_T_CLAMP = 1.0 - 1e-14
_C_ERF = 2.0 / math.sqrt(math.pi)


@dataclass(frozen=True)
class TimeGrid:
    """N grid points t_i = i*dt on [0, T], dt = T/(N-1), p+1 functions per step."""

    T: float
    N: int
    p: int

    def __post_init__(self) -> None:
        if not self.T > 0:
            raise ValueError(f"final time T must be positive, got {self.T}")
        if self.N < 3:
            raise ValueError(f"need at least 3 timesteps, got N={self.N}")
        if self.p < 0:
            raise ValueError(f"polynomial order must be >= 0, got p={self.p}")

    @property
    def dt(self) -> float:
        return self.T / (self.N - 1)

    @property
    def L(self) -> int:
        return self.N * (self.p + 1)

    def t(self, i: int) -> float:
        return i * self.dt

    def t_formal(self, i: int) -> float:
        """t_i with the conventions t_{-1} = t_0 = 0 and t_N = t_{N-1} = T."""
        j = 0 if i < 0 else (self.N - 1 if i > self.N - 1 else i)
        return j * self.dt


class TemporalBasisIndex(NamedTuple):
    flat: int
    timestep: int
    order: int


def flat_index(grid: TimeGrid, timestep: int, order: int) -> TemporalBasisIndex:
    if not 1 <= timestep <= grid.N:
        raise ValueError(f"timestep {timestep} outside 1..{grid.N}")
    if not 0 <= order <= grid.p:
        raise ValueError(f"order {order} outside 0..{grid.p}")
    return TemporalBasisIndex((timestep - 1) * (grid.p + 1) + order + 1, timestep, order)


def decode_flat(grid: TimeGrid, flat: int) -> TemporalBasisIndex:
    if not 1 <= flat <= grid.L:
        raise ValueError(f"flat index {flat} outside 1..{grid.L}")
    step, order = divmod(flat - 1, grid.p + 1)
    return TemporalBasisIndex(flat, step + 1, order)


def cutoff_f(t, deriv: int = 0):
    """Smooth step 0 -> 1 over [-1, 1] and its first two derivatives.

    f(t) = (1 + erf(2 artanh t)) / 2 inside, 0 left of -1, 1 right of +1.
    """
    if deriv not in (0, 1, 2):
        raise ValueError(f"deriv must be 0, 1 or 2, got {deriv}")
    t = np.asarray(t, dtype=float)
    scalar = t.ndim == 0
    t = np.atleast_1d(t)
    tc = np.minimum(np.maximum(t, -_T_CLAMP), _T_CLAMP)
    s = np.arctanh(tc)
    with np.errstate(under="ignore"):
        g = np.exp(-4.0 * s * s)
    if deriv == 0:
        val = 0.5 * erf(2.0 * s) + 0.5
        out = np.where(t >= 1.0, 1.0, val)
        out = np.where(t <= -1.0, 0.0, out)
    else:
        q = 1.0 - tc * tc
        if deriv == 1:
            val = _C_ERF * g / q
        else:
            val = _C_ERF * g * (2.0 * tc - 8.0 * s) / (q * q)
        out = np.where((np.abs(t) < 1.0) & (g > 0.0), val, 0.0)
    return float(out[0]) if scalar else out


def legendre_table(pmax: int, x):
    """P_m, P_m', P_m'' for m = 0..pmax by the Bonnet recurrence."""
    x = np.asarray(x, dtype=float)
    P = np.empty((pmax + 1,) + x.shape)
    D1 = np.empty_like(P)
    D2 = np.empty_like(P)
    P[0], D1[0], D2[0] = 1.0, 0.0, 0.0
    if pmax >= 1:
        P[1], D1[1], D2[1] = x, 1.0, 0.0
    for m in range(2, pmax + 1):
        a = (2 * m - 1) / m
        b = (m - 1) / m
        P[m] = a * x * P[m - 1] - b * P[m - 2]
        D1[m] = a * (P[m - 1] + x * D1[m - 1]) - b * D1[m - 2]
        D2[m] = a * (2.0 * D1[m - 1] + x * D2[m - 1]) - b * D2[m - 2]
    return P, D1, D2


def timestep_kind(grid: TimeGrid, timestep: int) -> str:
    if timestep == 1:
        return KIND_FIRST
    if timestep == grid.N:
        return KIND_LAST
    return KIND_INNER


def canonical_support(grid: TimeGrid, kind: str) -> float:
    return 2.0 * grid.dt if kind == KIND_INNER else grid.dt


def canonical_origin(grid: TimeGrid, timestep: int) -> float:
    """Time shift that maps b_{timestep, m} onto its canonical prototype."""
    kind = timestep_kind(grid, timestep)
    if kind == KIND_FIRST:
        return 0.0
    if kind == KIND_LAST:
        return grid.t(grid.N - 2)
    return grid.t(timestep - 2)


def support_interval(grid: TimeGrid, timestep: int) -> tuple[float, float]:
    o = canonical_origin(grid, timestep)
    return o, o + canonical_support(grid, timestep_kind(grid, timestep))


def _ramp(c: float, u, deriv: int):
    """f(c*u - 1) differentiated `deriv` times with respect to u."""
    return cutoff_f(c * u - 1.0, deriv) * c**deriv


def _inner_bump(dt: float, u, deriv: int):
    """rho on [0, 2dt]: rising ramp on [0, dt], falling ramp on [dt, 2dt]."""
    c = 2.0 / dt
    up = _ramp(c, u, deriv)
    if deriv == 0:
        down = 1.0 - _ramp(c, u - dt, 0)
    else:
        down = -_ramp(c, u - dt, deriv)
    out = np.where(u <= dt, up, down)
    out[(u <= 0.0) | (u >= 2.0 * dt)] = 0.0
    return out


def canonical_basis_all(grid: TimeGrid, kind: str, pmax: int, u, deriv: int = 0) -> np.ndarray:
    """All canonical prototypes of orders 0..pmax at offsets u (time derivative `deriv`).

    inner: rho(u) P_m(u/dt - 1) on [0, 2dt]
    last : f(2u/dt - 1) P_m(2u/dt - 1) on (0, dt]
    first: 8 (u/dt)^2 (1 - f(2u/dt - 1)) P_m(2u/dt - 1) on (0, dt)
    Shape (pmax+1,) + u.shape; exactly zero outside the support.
    """
    if deriv not in (0, 1, 2):
        raise ValueError(f"deriv must be 0, 1 or 2, got {deriv}")
    u = np.atleast_1d(np.asarray(u, dtype=float))
    dt = grid.dt
    if kind == KIND_INNER:
        P, P1, P2 = legendre_table(pmax, u / dt - 1.0)
        r0 = _inner_bump(dt, u, 0)
        if deriv == 0:
            out = r0 * P
        else:
            r1 = _inner_bump(dt, u, 1)
            if deriv == 1:
                out = r1 * P + r0 * P1 / dt
            else:
                r2 = _inner_bump(dt, u, 2)
                out = r2 * P + 2.0 * r1 * P1 / dt + r0 * P2 / dt**2
        out[:, (u <= 0.0) | (u >= 2.0 * dt)] = 0.0
        return out

    c = 2.0 / dt
    x = c * u - 1.0
    P, P1, P2 = legendre_table(pmax, x)
    if kind == KIND_LAST:
        f0 = cutoff_f(x, 0)
        if deriv == 0:
            out = f0 * P
        elif deriv == 1:
            out = c * (cutoff_f(x, 1) * P + f0 * P1)
        else:
            f1 = cutoff_f(x, 1)
            out = c * c * (cutoff_f(x, 2) * P + 2.0 * f1 * P1 + f0 * P2)
        out[:, (u <= 0.0) | (u > dt)] = 0.0
        return out
    if kind != KIND_FIRST:
        raise ValueError(f"unknown basis kind {kind!r}")
    # product rule on g(u) * q(u) * P(x(u)), g = 1 - f, q = (u/dt)^2
    g0 = 1.0 - cutoff_f(x, 0)
    g1 = -c * cutoff_f(x, 1)
    g2 = -c * c * cutoff_f(x, 2)
    q0 = (u / dt) ** 2
    q1 = 2.0 * u / dt**2
    q2 = 2.0 / dt**2
    if deriv == 0:
        out = 8.0 * g0 * q0 * P
    elif deriv == 1:
        out = 8.0 * (g1 * q0 * P + g0 * q1 * P + g0 * q0 * P1 * c)
    else:
        out = 8.0 * (
            g2 * q0 * P
            + g0 * q2 * P
            + g0 * q0 * P2 * c * c
            + 2.0 * g1 * q1 * P
            + 2.0 * g1 * q0 * P1 * c
            + 2.0 * g0 * q1 * P1 * c
        )
    out[:, (u <= 0.0) | (u >= dt)] = 0.0
    return out


def basis_b(grid: TimeGrid, idx, t, deriv: int = 0):
    """b_i(t) (or a time derivative) for a flat index or TemporalBasisIndex."""
    if isinstance(idx, (int, np.integer)):
        idx = decode_flat(grid, int(idx))
    t = np.asarray(t, dtype=float)
    scalar = t.ndim == 0
    u = np.atleast_1d(t) - canonical_origin(grid, idx.timestep)
    out = canonical_basis_all(grid, timestep_kind(grid, idx.timestep), idx.order, u, deriv)[idx.order]
    return float(out[0]) if scalar else out
