"""Krylov solvers for the block Hessenberg system on device vectors.

Reference interface (``tdbem.solvers``, /root/reference/pkg/src/tdbem/solvers.py):
  SolverConfig               :37-52
  DeflationState             :55-76 (M^-1 = I + U(|lambda| T^-1 - I)U^T)
  dense_schur / schur_eigenvalues / _smallest_invariant_basis  :79-126
  _orthonormal_extend        :129-142
  _run_restarted             :145-169
  _gmres_cycle_raw           :172-223 (MGS Arnoldi, Givens, restart)
  gmres / fgmres / dgmres    :226-273
  recursive_preconditioner   :276-315, _inner_cfg :318-320

Vectors of length n = L*M live on the device (torch float64 CUDA tensors; any
torch device works for the callback-only paths, which is how the CPU unit
tests exercise the Krylov logic).  The operator is a callback v -> A v on the
same device, normally BlockHessenbergMatrix.matvec (csrc/tdb_matvec.cu).  The
(m+1) x m Hessenberg matrix, Givens rotations, the triangular solve and the
Schur decompositions (at most 50 x 50) stay on the host, one small
device->host copy per Arnoldi step, exactly as the reference orders them.

The fixed-iteration inner solves of the recursive preconditioner (restart ==
max_iter, tol 1e-14: one cycle) take a host-sync-free path on CUDA vectors:
classical Gram-Schmidt with one re-orthogonalisation pass (two GEMVs per pass,
as accurate as the reference's MGS), and the Hessenberg / Givens / convergence
bookkeeping on the device (csrc/tdb_krylov.cu).  Early exit is emulated on the
device, so the iterate equals the one the reference's loop returns.  The whole
preconditioner application of a single-device solve is then captured once in
a CUDA graph and replayed per outer step.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla
import torch

__all__ = [
    "set_comm",
    "TorchDistComm",
    "SolverConfig",
    "DeflationState",
    "BreakdownError",
    "gmres",
    "dgmres",
    "fgmres",
    "recursive_preconditioner",
    "dense_schur",
    "schur_eigenvalues",
    "solve",
]


class BreakdownError(RuntimeError):
    """Arnoldi norm underflow without a converged residual."""


@dataclass
class SolverConfig:
    method: str = "gmres"
    restart: int = 50
    tol: float = 1e-5
    max_iter: int = 10000
    deflate_per_restart: int = 0
    max_deflation: int = 20
    recursion_depth: int = 0
    inner_iterations: tuple = ()

    def __post_init__(self):
        if self.restart < 1 or self.tol <= 0.0 or self.recursion_depth < 0:
            raise ValueError("invalid solver configuration")
        if not 0 <= self.deflate_per_restart <= self.max_deflation:
            raise ValueError("deflation counts must satisfy 0 <= l <= r")


class _LocalComm:
    """Single device: vectors are whole, reductions are no-ops."""

    size = 1
    capturable = True

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        return t


class TorchDistComm:
    """Row-block distributed vectors: every Krylov vector holds this
    rank's vertex rows for all time steps; dot products and norms are
    all-reduced (NCCL on CUDA tensors, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        # NCCL collectives can be captured in a CUDA graph (the preconditioner is
        # replayed as one graph per outer step); gloo ones cannot
        self.capturable = dist.get_backend(group) == "nccl"

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        if t.is_cuda and not self.capturable:  # gloo: host-staged
            c = t.cpu()
            self.dist.all_reduce(c, group=self.group)
            t.copy_(c)
            return t
        self.dist.all_reduce(t, group=self.group)
        return t


_COMM = _LocalComm()


def set_comm(comm) -> None:
    """Select the communicator used by every solver (None -> single device)."""
    global _COMM
    _COMM = comm if comm is not None else _LocalComm()


def _dot(u: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    return _COMM.allreduce_(torch.dot(u, v).reshape(1))[0]


def _norm(v: torch.Tensor) -> torch.Tensor:
    if _COMM.size == 1:
        return torch.linalg.vector_norm(v)
    return torch.sqrt(_COMM.allreduce_(torch.dot(v, v).reshape(1))[0])


class DeflationState:
    """Approximate invariant subspace U (n, r) with AU = A U; M^-1 applied on the device."""

    def __init__(self, U: torch.Tensor, AU: torch.Tensor, lambda_max: float = 0.0):
        self.U = U
        self.AU = AU
        self.lambda_max = lambda_max
        self._lu = None

    @property
    def rank(self) -> int:
        return self.U.shape[1]

    def t_small(self) -> np.ndarray:
        return _COMM.allreduce_((self.U.T @ self.AU).contiguous()).cpu().numpy()

    def apply_minv(self, v: torch.Tensor) -> torch.Tensor:
        if self.rank == 0:
            return v
        if self._lu is None:
            self._lu = sla.lu_factor(self.t_small())
        w = _COMM.allreduce_((self.U.T @ v).contiguous())
        y = sla.lu_solve(self._lu, w.cpu().numpy())
        y = torch.as_tensor(y, dtype=v.dtype, device=v.device)
        return v + self.U @ (self.lambda_max * y - w)

    def _invalidate(self):
        self._lu = None


def dense_schur(H: np.ndarray):
    T, Q = sla.schur(np.asarray(H, dtype=float), output="real")
    return Q, T


def schur_eigenvalues(T: np.ndarray) -> np.ndarray:
    n = T.shape[0]
    vals = np.empty(n, dtype=complex)
    i = 0
    while i < n:
        if i + 1 < n and abs(T[i + 1, i]) > 0.0:
            a, b, c, d = T[i, i], T[i, i + 1], T[i + 1, i], T[i + 1, i + 1]
            tr, det = a + d, a * d - b * c
            root = np.sqrt(complex(tr * tr / 4.0 - det))
            vals[i], vals[i + 1] = tr / 2.0 + root, tr / 2.0 - root
            i += 2
        else:
            vals[i] = T[i, i]
            i += 1
    return vals


def _smallest_invariant_basis(H: np.ndarray, l: int):
    """Schur basis of the l smallest-modulus eigenvalues of H (+1 if a conjugate pair straddles)."""
    Q, T = dense_schur(H)
    vals = schur_eigenvalues(T)
    lam_max = float(np.max(np.abs(vals)))
    if l <= 0:
        return np.zeros((H.shape[0], 0)), lam_max
    n = len(vals)
    if l >= n:
        return Q, lam_max
    mods = np.sort(np.abs(vals))
    thr = 0.5 * (mods[l - 1] + mods[l]) if mods[l] > mods[l - 1] else mods[l - 1] * (1 + 1e-12)
    _, QQ, sdim = sla.schur(np.asarray(H, dtype=float), output="real",
                            sort=lambda re, im: np.hypot(re, im) <= thr)
    return QQ[:, :sdim], lam_max


def _orthonormal_extend(U: torch.Tensor, W: torch.Tensor, drop_tol: float = 1e-12) -> torch.Tensor:
    """Append columns of W to U: MGS with one reorthogonalisation pass."""
    cols = [U[:, j] for j in range(U.shape[1])]
    for j in range(W.shape[1]):
        w = W[:, j].clone()
        for _ in range(2):
            for u in cols:
                w = w - _dot(u, w) * u
        nw = float(_norm(w))
        if nw > drop_tol:
            cols.append(w / nw)
    if not cols:
        return torch.zeros((U.shape[0], 0), dtype=U.dtype, device=U.device)
    return torch.stack(cols, dim=1)


def _gmres_cycle_raw(apply_A, b, x0, m, tol_abs, precond, history):
    """One restart cycle (reference solvers.py:172-223) with device vectors."""
    n = b.shape[0]
    dev, dt = b.device, b.dtype
    r0 = b - apply_A(x0)
    beta = float(_norm(r0))
    if beta <= tol_abs:
        history.append(beta)
        return x0, True, False, dict(k=0)
    V = torch.zeros((m + 1, n), dtype=dt, device=dev)
    Z = V[:m] if precond is None else torch.zeros((m, n), dtype=dt, device=dev)
    H = np.zeros((m + 1, m))
    Hraw = np.zeros((m + 1, m))
    cs = np.zeros(m)
    sn = np.zeros(m)
    g = np.zeros(m + 1)
    g[0] = beta
    V[0] = r0 / beta
    hcol = torch.zeros(m + 1, dtype=dt, device=dev)
    k_done = 0
    breakdown = False
    for k in range(m):
        if precond is None:
            z = V[k]
        else:
            z = precond(V[k])
            Z[k] = z
        w = apply_A(z).clone()
        if w.is_cuda and _COMM.size == 1 and k < 63 and w.dtype == torch.float64:
            # CGS2 orthogonalisation + norm on the device (tdb_krylov_arnoldi)
            from . import _lib

            _lib.check(_lib.LIB.tdb_krylov_arnoldi(_ptr(V), n, n, k, _ptr(w), _ptr(hcol), None, None, 0, None,
                                                   None, None, None,
                                                   C_void(torch.cuda.current_stream(dev).cuda_stream)),
                       "krylov_arnoldi")
        elif _COMM.size > 1:
            # row-block distributed vectors: classical Gram-Schmidt with one re-orthogonalisation
            # pass, each pass ONE batched all-reduce of the k+1 coefficients, then
            # the norm: 3 collectives per Arnoldi step instead of k+2 for MGS
            Vk = V[: k + 1]
            h = _gemv_t(Vk, w)
            w.sub_(torch.mv(Vk.T, h))
            h2 = _gemv_t(Vk, w)
            w.sub_(torch.mv(Vk.T, h2))
            torch.add(h, h2, out=hcol[: k + 1])
            hcol[k + 1] = _norm(w)
        else:
            # modified Gram-Schmidt: h_j computed and subtracted one vector at a time
            # (the reference's order, solvers.py:194-198)
            for j in range(k + 1):
                torch.dot(V[j], w, out=hcol[j])
                w.addcmul_(V[j], hcol[j : j + 1], value=-1.0)
            hcol[k + 1] = _norm(w)
        col = hcol[: k + 2].cpu().numpy()
        H[: k + 2, k] = col
        Hraw[: k + 2, k] = col
        hk = H[k + 1, k]
        for j in range(k):
            t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
            H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
            H[j, k] = t
        denom = np.hypot(H[k, k], H[k + 1, k])
        cs[k] = H[k, k] / denom if denom > 0 else 1.0
        sn[k] = H[k + 1, k] / denom if denom > 0 else 0.0
        H[k, k] = denom
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k] * g[k]
        H[k + 1, k] = 0.0
        k_done = k + 1
        history.append(abs(g[k + 1]))
        if abs(g[k + 1]) <= tol_abs:
            break
        if hk <= 1e-14 * beta:
            breakdown = True
            break
        V[k + 1] = w / hk
    y = sla.solve_triangular(H[:k_done, :k_done], g[:k_done], lower=False)
    yd = torch.as_tensor(y, dtype=dt, device=dev)
    x = x0 + Z[:k_done].T @ yd
    converged = history[-1] <= tol_abs
    return x, converged, breakdown, dict(V=V, Hraw=Hraw, k=k_done)


def _gemv_t(V: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """h = V w (rows of V are Krylov vectors), all-reduced across row blocks."""
    h = torch.mv(V, w)
    return _COMM.allreduce_(h) if _COMM.size > 1 else h


def _cycle_fixed_device(apply_A, b: torch.Tensor, m: int, tol: float, precond, err: torch.Tensor):
    """One GMRES / FGMRES cycle of at most m steps from x0 = 0 with no host
    synchronisation (the reference's _run_restarted with restart == max_iter,
    solvers.py:145-169 + :172-223).  Returns x; a breakdown without convergence
    sets err[0] = 1 (BreakdownError, checked by the caller)."""
    from . import _lib

    n = b.shape[0]
    dev, dt = b.device, b.dtype
    stream = C_void(torch.cuda.current_stream(dev).cuda_stream)
    st = torch.empty(_lib.KS_NSTATE, dtype=dt, device=dev)
    H = torch.zeros((m + 1, m), dtype=dt, device=dev)
    cs = torch.empty(m, dtype=dt, device=dev)
    sn = torch.empty(m, dtype=dt, device=dev)
    g = torch.zeros(m + 1, dtype=dt, device=dev)
    hcol = torch.empty(m + 1, dtype=dt, device=dev)
    V = torch.empty((m, n), dtype=dt, device=dev)
    if n == 0:
        return torch.zeros_like(b)
    Z = V if precond is None else torch.empty((m, n), dtype=dt, device=dev)
    beta = _norm(b).reshape(1)
    L = _lib.LIB
    _lib.check(L.tdb_krylov_init(_ptr(st), _ptr(beta), float(tol), _ptr(g), stream), "krylov_init")
    torch.div(b, beta, out=V[0])
    fused = _COMM.size == 1 and m < 64
    for k in range(m):
        if precond is not None:
            Z[k].copy_(precond(V[k]))
        w = apply_A(Z[k])
        if fused:  # CGS2 + norm + Givens + V[k+1] = w / ||w|| (tdb_krylov_arnoldi)
            vnext = _ptr(V[k + 1]) if k + 1 < m else None
            _lib.check(L.tdb_krylov_arnoldi(_ptr(V), n, n, k, _ptr(w), _ptr(hcol), _ptr(st), _ptr(H), m, _ptr(cs),
                                            _ptr(sn), _ptr(g), vnext, stream), "krylov_arnoldi")
            continue
        w = w.clone()
        Vk = V[: k + 1]
        h = _gemv_t(Vk, w)
        w.sub_(torch.mv(Vk.T, h))
        h2 = _gemv_t(Vk, w)
        w.sub_(torch.mv(Vk.T, h2))
        torch.add(h, h2, out=hcol[: k + 1])
        hcol[k + 1 : k + 2].copy_(_norm(w).reshape(1))
        _lib.check(L.tdb_krylov_givens(_ptr(st), k, _ptr(hcol), _ptr(H), m, _ptr(cs), _ptr(sn), _ptr(g),
                                       stream), "krylov_givens")
        if k + 1 < m:
            torch.div(w, hcol[k + 1 : k + 2], out=V[k + 1])
    x = torch.empty(n, dtype=dt, device=dev)
    _lib.check(L.tdb_krylov_update(_ptr(x), None, _ptr(Z), n, n, _ptr(st), _ptr(H), m, _ptr(g), m, stream),
               "krylov_update")
    _lib.check(L.tdb_krylov_flag(_ptr(st), _ptr(err), stream), "krylov_flag")
    return x


def C_void(v):
    import ctypes

    return ctypes.c_void_p(v)


def _ptr(t: torch.Tensor):
    return C_void(t.data_ptr())


def _run_restarted(apply_A, b, cfg: SolverConfig, precond_factory, per_cycle=None):
    nb = float(_norm(b))
    if nb == 0.0:
        return torch.zeros_like(b), [0.0]
    tol_abs = cfg.tol * nb
    x = torch.zeros_like(b)
    history: list = []
    while len(history) < cfg.max_iter:
        m = min(cfg.restart, cfg.max_iter - len(history))
        precond = precond_factory()
        x, converged, breakdown, raw = _gmres_cycle_raw(apply_A, b, x, m, tol_abs, precond, history)
        if per_cycle is not None and raw["k"] > 0:
            per_cycle(raw)
        if converged:
            break
        if breakdown:
            raise BreakdownError("Arnoldi breakdown before convergence")
    return x, [h / nb for h in history]


def gmres(apply_A, b, cfg: SolverConfig):
    """Restarted GMRES(m); returns (x, relative residual history)."""
    return _run_restarted(apply_A, b, cfg, lambda: None)


def fgmres(apply_A, b, cfg: SolverConfig, precond=None):
    """Flexible GMRES with a right preconditioner callback that may vary."""
    factory = (lambda: None) if precond is None else (lambda: precond)
    return _run_restarted(apply_A, b, cfg, factory)


def dgmres(apply_A, b, cfg: SolverConfig):
    """Deflated restarted GMRES(m, l); returns (x, history, DeflationState)."""
    n = b.shape[0]
    state = DeflationState(U=torch.zeros((n, 0), dtype=b.dtype, device=b.device),
                           AU=torch.zeros((n, 0), dtype=b.dtype, device=b.device))

    def factory():
        return None if state.rank == 0 else state.apply_minv

    def per_cycle(raw):
        k = raw["k"]
        if cfg.deflate_per_restart <= 0 or state.rank >= cfg.max_deflation:
            if k > 0:
                vals = np.abs(schur_eigenvalues(dense_schur(raw["Hraw"][:k, :k])[1]))
                state.lambda_max = max(state.lambda_max, float(vals.max()))
                state._invalidate()
            return
        S, lam = _smallest_invariant_basis(raw["Hraw"][:k, :k], cfg.deflate_per_restart)
        state.lambda_max = max(state.lambda_max, lam)
        state._invalidate()
        if S.shape[1] == 0:
            return
        Sd = torch.as_tensor(S, dtype=b.dtype, device=b.device)
        W = raw["V"][:k].T @ Sd
        U_new = _orthonormal_extend(state.U, W)
        if U_new.shape[1] > cfg.max_deflation:
            U_new = U_new[:, : cfg.max_deflation]
        added = U_new[:, state.rank :]
        if added.shape[1]:
            AU_add = torch.stack([apply_A(added[:, j].contiguous()) for j in range(added.shape[1])], dim=1)
            state.U = U_new
            state.AU = torch.cat([state.AU, AU_add], dim=1)

    x, history = _run_restarted(apply_A, b, cfg, factory, per_cycle)
    return x, history, state


def _inner_cfg(cfg: SolverConfig, level: int) -> SolverConfig:
    iters = cfg.inner_iterations[level - 1] if level <= len(cfg.inner_iterations) else 10
    return SolverConfig(method="fgmres", restart=iters, tol=1e-14, max_iter=iters)


class _ErrBox:
    """Sticky device breakdown flag shared by the inner solves of one preconditioner."""

    def __init__(self):
        self.t = None

    def on(self, device) -> torch.Tensor:
        if self.t is None or self.t.device != device:
            self.t = torch.zeros(1, dtype=torch.float64, device=device)
        return self.t


def _inner_solve(apply_A, r, icfg: SolverConfig, precond, err: _ErrBox):
    """Fixed-iteration inner FGMRES (one cycle): device path on CUDA vectors."""
    if r.is_cuda:
        return _cycle_fixed_device(apply_A, r, icfg.restart, icfg.tol, precond, err.on(r.device))
    x, _ = fgmres(apply_A, r, icfg, precond=precond)
    return x


class _GraphedPreconditioner:
    """r -> P r of the recursive preconditioner, captured once in a CUDA graph after
    two eager warm-up calls (which create every matvec plan and communicator).  With
    row-block distributed vectors the capture includes the NCCL all-gathers and
    all-reduces (comm.capturable); a gloo communicator stays eager."""

    def __init__(self, fn, err: _ErrBox):
        self.fn = fn
        self.err = err
        self.calls = 0
        self.graph = None
        self.static_in = self.static_out = None

    def _check(self):
        if self.err.t is not None and float(self.err.t[0]) != 0.0:
            raise BreakdownError("inner Arnoldi breakdown before convergence")

    def __call__(self, r):
        if not r.is_cuda:
            return self.fn(r)
        self.calls += 1
        if not getattr(_COMM, "capturable", _COMM.size == 1) or self.calls <= 2:
            out = self.fn(r)
            self._check()
            return out
        if self.graph is None:
            self.static_in = r.clone()
            torch.cuda.synchronize(r.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.static_out = self.fn(self.static_in)
            self.graph = g
        self.static_in.copy_(r)
        self.graph.replay()
        self._check()
        return self.static_out.clone()


def recursive_preconditioner(A, cfg: SolverConfig, level: int = 1, rows=None, err=None):
    """Block lower-triangular half-split preconditioner (paper 4.2, reference :276-315).

    A.matvec(v, rows, cols) is the device block Hessenberg matvec; each half is
    solved with i_level FGMRES steps, preconditioned one level deeper while
    level < m_r.
    """
    lo, hi = rows if rows is not None else (1, A.grid.N)
    top = err is None
    if top:
        err = _ErrBox()
    count = hi - lo + 1
    if count < 2:
        def solo(r):
            return _inner_solve(lambda v: A.matvec(v, rows=(lo, hi), cols=(lo, hi)), r, _inner_cfg(cfg, level),
                                None, err)
        return _GraphedPreconditioner(solo, err) if top else solo
    split = lo + (count + 1) // 2 - 1
    n1 = (split - lo + 1) * (A.grid.p + 1) * A.M
    inner_1 = inner_2 = None
    if level < cfg.recursion_depth:
        inner_1 = recursive_preconditioner(A, cfg, level + 1, rows=(lo, split), err=err)
        inner_2 = recursive_preconditioner(A, cfg, level + 1, rows=(split + 1, hi), err=err)

    def half_solve(r, blo, bhi, prec):
        return _inner_solve(lambda v: A.matvec(v, rows=(blo, bhi), cols=(blo, bhi)), r, _inner_cfg(cfg, level),
                            prec, err)

    def prec(r):
        r1 = r[:n1].contiguous()
        r2 = r[n1:]
        x1 = half_solve(r1, lo, split, inner_1)
        r2c = r2 - A.matvec(x1.contiguous(), rows=(split + 1, hi), cols=(lo, split))
        x2 = half_solve(r2c.contiguous(), split + 1, hi, inner_2)
        return torch.cat([x1, x2])

    return _GraphedPreconditioner(prec, err) if top else prec


def solve(A, b, cfg: SolverConfig, device=None):
    """Convenience driver mirroring the reference CLI's _solve (cli.py:166-177):
    method 'gmres' | 'dgmres' | 'fgmres-recursive'.  b numpy or device tensor."""
    is_np = not isinstance(b, torch.Tensor)
    if is_np:
        dev = device if device is not None else torch.device("cuda", A._dev.ctx.device if A._dev else 0)
        bd = torch.as_tensor(np.ascontiguousarray(b, dtype=np.float64)).to(dev)
    else:
        bd = b
    apply_A = lambda v: A.matvec(v.contiguous())
    if cfg.method == "gmres":
        x, hist = gmres(apply_A, bd, cfg)
    elif cfg.method == "dgmres":
        x, hist, _ = dgmres(apply_A, bd, cfg)
    else:
        x, hist = fgmres(apply_A, bd, cfg, precond=recursive_preconditioner(A, cfg))
    return (x.cpu().numpy() if is_np else x), hist
