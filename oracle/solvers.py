"""ORACLE (test infrastructure): numpy restatement of the reference Krylov solvers.

Follows /root/reference/pkg/src/tdbem/solvers.py function by function:
  _cycle        <- _gmres_cycle_raw :172-223 (MGS Arnoldi + Givens)
  _restarted    <- _run_restarted   :145-169
  gmres/fgmres/dgmres               :226-273
  recursive_preconditioner          :276-315, _inner_cfg :318-320
  smallest_invariant_basis          :105-126
Used only by tests/ to check the device solvers (paper_1503_07221_b200.solvers).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla


class Breakdown(RuntimeError):
    pass


class Cfg:
    def __init__(self, restart=50, tol=1e-5, max_iter=10000, deflate_per_restart=0, max_deflation=20,
                 recursion_depth=0, inner_iterations=()):
        self.restart, self.tol, self.max_iter = restart, tol, max_iter
        self.deflate_per_restart, self.max_deflation = deflate_per_restart, max_deflation
        self.recursion_depth, self.inner_iterations = recursion_depth, tuple(inner_iterations)


def _cycle(A, b, x0, m, tol_abs, M, hist):
    n = len(b)
    r0 = b - A(x0)
    beta = np.linalg.norm(r0)
    if beta <= tol_abs:
        hist.append(beta)
        return x0, True, False, {"k": 0}
    V = np.zeros((n, m + 1))
    Z = np.zeros((n, m))
    H = np.zeros((m + 1, m))
    Hr = np.zeros((m + 1, m))
    c = np.zeros(m)
    s = np.zeros(m)
    g = np.zeros(m + 1)
    g[0] = beta
    V[:, 0] = r0 / beta
    kk = 0
    brk = False
    for k in range(m):
        z = V[:, k] if M is None else M(V[:, k])
        Z[:, k] = z
        w = A(z)
        for j in range(k + 1):
            H[j, k] = V[:, j] @ w
            w = w - H[j, k] * V[:, j]
        H[k + 1, k] = np.linalg.norm(w)
        Hr[: k + 2, k] = H[: k + 2, k]
        hk = H[k + 1, k]
        for j in range(k):
            t = c[j] * H[j, k] + s[j] * H[j + 1, k]
            H[j + 1, k] = -s[j] * H[j, k] + c[j] * H[j + 1, k]
            H[j, k] = t
        d = np.hypot(H[k, k], H[k + 1, k])
        c[k] = H[k, k] / d if d > 0 else 1.0
        s[k] = H[k + 1, k] / d if d > 0 else 0.0
        H[k, k] = d
        g[k + 1] = -s[k] * g[k]
        g[k] = c[k] * g[k]
        H[k + 1, k] = 0.0
        kk = k + 1
        hist.append(abs(g[k + 1]))
        if abs(g[k + 1]) <= tol_abs:
            break
        if hk <= 1e-14 * beta:
            brk = True
            break
        V[:, k + 1] = w / hk
    y = sla.solve_triangular(H[:kk, :kk], g[:kk], lower=False)
    return x0 + Z[:, :kk] @ y, hist[-1] <= tol_abs, brk, {"V": V, "Hraw": Hr, "k": kk}


def _restarted(A, b, cfg, factory, per_cycle=None):
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return np.zeros_like(b), [0.0]
    tol_abs = cfg.tol * nb
    x = np.zeros_like(b)
    hist = []
    while len(hist) < cfg.max_iter:
        m = min(cfg.restart, cfg.max_iter - len(hist))
        x, conv, brk, raw = _cycle(A, b, x, m, tol_abs, factory(), hist)
        if per_cycle is not None and raw["k"] > 0:
            per_cycle(raw)
        if conv:
            break
        if brk:
            raise Breakdown("Arnoldi breakdown")
    return x, [h / nb for h in hist]


def gmres(A, b, cfg):
    return _restarted(A, b, cfg, lambda: None)


def fgmres(A, b, cfg, M=None):
    return _restarted(A, b, cfg, lambda: M)


def _schur_eigs(T):
    n = T.shape[0]
    out = np.empty(n, dtype=complex)
    i = 0
    while i < n:
        if i + 1 < n and abs(T[i + 1, i]) > 0.0:
            a, b_, c_, d = T[i, i], T[i, i + 1], T[i + 1, i], T[i + 1, i + 1]
            tr, det = a + d, a * d - b_ * c_
            rt = np.sqrt(complex(tr * tr / 4.0 - det))
            out[i], out[i + 1] = tr / 2 + rt, tr / 2 - rt
            i += 2
        else:
            out[i] = T[i, i]
            i += 1
    return out


def smallest_invariant_basis(H, l):
    T, Q = sla.schur(H, output="real")
    vals = _schur_eigs(T)
    lam = float(np.max(np.abs(vals)))
    if l <= 0:
        return np.zeros((H.shape[0], 0)), lam
    if l >= len(vals):
        return Q, lam
    mods = np.sort(np.abs(vals))
    thr = 0.5 * (mods[l - 1] + mods[l]) if mods[l] > mods[l - 1] else mods[l - 1] * (1 + 1e-12)
    _, QQ, sdim = sla.schur(H, output="real", sort=lambda re, im: np.hypot(re, im) <= thr)
    return QQ[:, :sdim], lam


def dgmres(A, b, cfg):
    n = len(b)
    st = {"U": np.zeros((n, 0)), "AU": np.zeros((n, 0)), "lam": 0.0}

    def minv(v):
        U, AU = st["U"], st["AU"]
        w = U.T @ v
        y = sla.lu_solve(sla.lu_factor(U.T @ AU), w)
        return v + U @ (st["lam"] * y - w)

    def factory():
        return None if st["U"].shape[1] == 0 else minv

    def per_cycle(raw):
        k = raw["k"]
        r = st["U"].shape[1]
        if cfg.deflate_per_restart <= 0 or r >= cfg.max_deflation:
            T = sla.schur(raw["Hraw"][:k, :k], output="real")[0]
            st["lam"] = max(st["lam"], float(np.abs(_schur_eigs(T)).max()))
            return
        S, lam = smallest_invariant_basis(raw["Hraw"][:k, :k], cfg.deflate_per_restart)
        st["lam"] = max(st["lam"], lam)
        if S.shape[1] == 0:
            return
        W = raw["V"][:, :k] @ S
        cols = [st["U"][:, j] for j in range(r)]
        for j in range(W.shape[1]):
            w = W[:, j].copy()
            for _ in range(2):
                for u in cols:
                    w -= (u @ w) * u
            nw = np.linalg.norm(w)
            if nw > 1e-12:
                cols.append(w / nw)
        Un = np.column_stack(cols)[:, : cfg.max_deflation] if cols else np.zeros((n, 0))
        add = Un[:, r:]
        if add.shape[1]:
            st["AU"] = np.hstack([st["AU"], np.column_stack([A(add[:, j]) for j in range(add.shape[1])])])
            st["U"] = Un

    x, hist = _restarted(A, b, cfg, factory, per_cycle)
    return x, hist, st


def _inner(cfg, level):
    it = cfg.inner_iterations[level - 1] if level <= len(cfg.inner_iterations) else 10
    return Cfg(restart=it, tol=1e-14, max_iter=it)


def recursive_preconditioner(matvec, N, block, cfg, level=1, rows=None):
    """matvec(x, rows, cols); block = (p+1) M entries per time step."""
    lo, hi = rows if rows is not None else (1, N)
    cnt = hi - lo + 1
    if cnt < 2:
        return lambda r: fgmres(lambda v: matvec(v, (lo, hi), (lo, hi)), r, _inner(cfg, level))[0]
    split = lo + (cnt + 1) // 2 - 1
    n1 = (split - lo + 1) * block
    p1 = p2 = None
    if level < cfg.recursion_depth:
        p1 = recursive_preconditioner(matvec, N, block, cfg, level + 1, (lo, split))
        p2 = recursive_preconditioner(matvec, N, block, cfg, level + 1, (split + 1, hi))

    def half(r, a, b_, M):
        return fgmres(lambda v: matvec(v, (a, b_), (a, b_)), r, _inner(cfg, level), M)[0]

    def prec(r):
        x1 = half(r[:n1], lo, split, p1)
        r2 = r[n1:] - matvec(x1, (split + 1, hi), (lo, split))
        return np.concatenate([x1, half(r2, split + 1, hi, p2)])

    return prec
