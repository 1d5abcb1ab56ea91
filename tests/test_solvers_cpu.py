"""Krylov solver logic (device code run on CPU torch tensors) vs the oracle and the
reference's golden solutions; mirrors reference tests/test_solvers.py."""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import solvers as OS
from paper_1503_07221_b200.solvers import (
    BreakdownError,
    SolverConfig,
    dense_schur,
    dgmres,
    fgmres,
    gmres,
    recursive_preconditioner,
    schur_eigenvalues,
)
from paper_1503_07221_b200.temporal_basis import TimeGrid


def T(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64))


class DenseBlockOp:
    """BlockHessenbergMatrix stand-in over a dense matrix (for the solver logic only)."""

    def __init__(self, dense, grid, M):
        self.D = T(dense)
        self.grid, self.M = grid, M
        self.blk = (grid.p + 1) * M

    def matvec(self, x, rows=None, cols=None):
        rlo, rhi = rows if rows is not None else (1, self.grid.N)
        clo, chi = cols if cols is not None else (1, self.grid.N)
        sub = self.D[(rlo - 1) * self.blk : rhi * self.blk, (clo - 1) * self.blk : chi * self.blk]
        return sub @ x


def well_conditioned(n=200, seed=0):
    rng = np.random.default_rng(seed)
    return np.eye(n) + (0.5 / np.sqrt(n)) * rng.standard_normal((n, n)), rng.standard_normal(n)


def test_config_validation():
    with pytest.raises(ValueError):
        SolverConfig(restart=0)
    with pytest.raises(ValueError):
        SolverConfig(tol=0.0)
    with pytest.raises(ValueError):
        SolverConfig(deflate_per_restart=5, max_deflation=3)
    with pytest.raises(ValueError):
        SolverConfig(recursion_depth=-1)


def test_schur_helpers():
    rng = np.random.default_rng(5)
    H = rng.standard_normal((20, 20))
    Q, Tm = dense_schur(H)
    assert np.linalg.norm(Q @ Tm @ Q.T - H) < 1e-12 * np.linalg.norm(H)
    got = np.sort_complex(schur_eigenvalues(dense_schur(H[:15, :15])[1]))
    assert np.max(np.abs(got - np.sort_complex(np.linalg.eigvals(H[:15, :15])))) < 1e-10


def test_gmres_random_vs_reference_golden():
    g = golden("solvers.npz")
    A, b = g["rand_A"], g["rand_b"]
    x, hist = gmres(lambda v: T(A) @ v, T(b), SolverConfig(restart=50, tol=1e-12))
    assert len(hist) == len(g["rand_gmres_hist"])
    assert np.allclose(hist, g["rand_gmres_hist"], rtol=1e-6, atol=1e-14)
    assert np.linalg.norm(x.numpy() - g["rand_gmres_x"]) < 1e-10 * np.linalg.norm(g["rand_gmres_x"])
    x, hist, st = dgmres(lambda v: T(A) @ v, T(b), SolverConfig(restart=20, tol=1e-12, deflate_per_restart=2,
                                                                max_deflation=8))
    assert np.linalg.norm(x.numpy() - g["rand_dgm_x"]) < 1e-10 * np.linalg.norm(g["rand_dgm_x"])
    assert 0 <= st.rank <= 8


def test_identity_zero_and_breakdown():
    b = T(np.arange(1.0, 9.0))
    x, hist = gmres(lambda v: v, b, SolverConfig(tol=1e-12))
    assert np.allclose(x.numpy(), b.numpy()) and len(hist) == 1
    x, hist = gmres(lambda v: v, T(np.zeros(5)), SolverConfig())
    assert torch.all(x == 0)
    A = T(np.outer(np.ones(6), np.ones(6)))
    with pytest.raises(BreakdownError):
        gmres(lambda v: A @ v, T(np.arange(1.0, 7.0)), SolverConfig(restart=6, tol=1e-12, max_iter=12))


def test_exact_deflation_spectrum():
    d = np.full(40, 10.0)
    d[0] = 2.0
    A = T(np.diag(d))
    b = T(np.random.default_rng(2).standard_normal(40))
    x, hist, st = dgmres(lambda v: A @ v, b, SolverConfig(restart=10, tol=1e-13, deflate_per_restart=1,
                                                          max_deflation=4))
    assert np.linalg.norm((A @ x - b).numpy()) <= 1e-12 * np.linalg.norm(b.numpy())
    assert st.rank >= 1 and np.abs(st.U[0, :].numpy()).max() > 0.99
    assert st.lambda_max == pytest.approx(10.0, rel=1e-6)


def test_fgmres_identity_and_exact_inverse():
    A, b = well_conditioned(seed=4)
    cfg = SolverConfig(restart=30, tol=1e-12)
    xg, hg = gmres(lambda v: T(A) @ v, T(b), cfg)
    xf, hf = fgmres(lambda v: T(A) @ v, T(b), cfg, precond=lambda v: v.clone())
    assert np.max(np.abs((xg - xf).numpy())) < 1e-13
    Ai = T(np.linalg.inv(A))
    x, hist = fgmres(lambda v: T(A) @ v, T(b), SolverConfig(restart=10, tol=1e-12), precond=lambda v: Ai @ v)
    assert len(hist) <= 3


def test_l_zero_identical_to_gmres():
    A, b = well_conditioned(seed=3)
    xg, hg = gmres(lambda v: T(A) @ v, T(b), SolverConfig(restart=25, tol=1e-12))
    xd, hd, st = dgmres(lambda v: T(A) @ v, T(b), SolverConfig(restart=25, tol=1e-12, deflate_per_restart=0))
    assert torch.equal(xg, xd) and hg == hd and st.rank == 0


def test_recursive_preconditioner_vs_reference_golden():
    g = golden("solvers.npz")
    dense = golden("blocks_two_tri_N6_p1.npz")["dense"]
    grid = TimeGrid(T=3.0, N=6, p=1)
    op = DenseBlockOp(dense, grid, 4)
    b = T(g["b9"])
    cfg = SolverConfig(restart=40, tol=1e-8, max_iter=2000, recursion_depth=2, inner_iterations=(2, 6))
    x, hist = fgmres(lambda v: op.matvec(v), b, cfg, precond=recursive_preconditioner(op, cfg))
    # the flexible inner solves amplify 1e-16 differences: the reference itself needs 74
    # (block matvec) or 75 (dense matvec) outer steps here, so iteration counts are not
    # compared; the first steps and the converged solutions are.
    assert np.allclose(hist[:4], g["frec_hist"][:4], rtol=1e-9)
    assert hist[-1] <= 1e-8
    xd = np.linalg.solve(dense, g["b9"])
    assert np.linalg.norm(x.numpy() - xd) <= 1e-5 * np.linalg.norm(xd)
    cfg = SolverConfig(restart=40, tol=1e-12, max_iter=4000, recursion_depth=2, inner_iterations=(2, 6))
    x, hist = fgmres(lambda v: op.matvec(v), b, cfg, precond=recursive_preconditioner(op, cfg))
    assert np.linalg.norm(x.numpy() - g["frec12_x"]) <= 1e-8 * np.linalg.norm(g["frec12_x"])
    assert np.linalg.norm(dense @ x.numpy() - g["b9"]) <= 1e-11 * np.linalg.norm(g["b9"])


def test_oracle_solvers_vs_reference_golden():
    g = golden("solvers.npz")
    dense = golden("blocks_two_tri_N6_p1.npz")["dense"]
    blk = 8
    mv = lambda x, rows, cols: dense[(rows[0] - 1) * blk : rows[1] * blk, (cols[0] - 1) * blk : cols[1] * blk] @ x
    cfg = OS.Cfg(restart=40, tol=1e-8, max_iter=2000, recursion_depth=2, inner_iterations=(2, 6))
    x, hist = OS.fgmres(lambda v: dense @ v, g["b9"], cfg, OS.recursive_preconditioner(mv, 6, blk, cfg))
    assert np.allclose(hist[:4], g["frec_hist"][:4], rtol=1e-9) and hist[-1] <= 1e-8
    x, hist = OS.gmres(lambda v: dense @ v, g["b9"], OS.Cfg(restart=40, tol=1e-8, max_iter=2000))
    assert len(hist) == len(g["gmres_hist"])
    x, hist, st = OS.dgmres(lambda v: dense @ v, g["b9"], OS.Cfg(restart=20, tol=1e-12, max_iter=4000,
                                                                deflate_per_restart=2, max_deflation=8))
    assert np.linalg.norm(x - g["dgm_x"]) <= 1e-8 * np.linalg.norm(g["dgm_x"])


def test_two_tri_recursive_iteration_count_is_roundoff_chaotic():
    """Why the device FGMRES takes 40 outer steps on two_tri (N=6, p=1, 2(2,6)) where the reference
    takes 74: the inner fixed 6-step solves on 8-16 unknowns run into near-breakdown (w / h_k+1,k
    with h tiny), so the preconditioner carries roundoff amplified to ~1e-8 within 7 outer steps.
    The reference algorithm itself (oracle restatement, MGS like ref solvers.py:172-223) lands
    anywhere in a wide band when every matvec is perturbed by 1e-16 relative (the reference gives
    74 with its block matvec, 75 with a dense one); solutions agree to the solver tolerance."""
    g = golden("solvers.npz")
    dense = golden("blocks_two_tri_N6_p1.npz")["dense"]
    blk = 8
    counts = []
    for seed in range(16):
        rng = np.random.default_rng(seed)
        pert = lambda y: y * (1.0 + 1e-16 * rng.standard_normal(len(y)))
        mv = lambda x, rows, cols: pert(dense[(rows[0] - 1) * blk:rows[1] * blk,
                                              (cols[0] - 1) * blk:cols[1] * blk] @ x)
        cfg = OS.Cfg(restart=40, tol=1e-8, max_iter=2000, recursion_depth=2, inner_iterations=(2, 6))
        x, hist = OS.fgmres(lambda v: pert(dense @ v), g["b9"], cfg, OS.recursive_preconditioner(mv, 6, blk, cfg))
        assert hist[-1] <= 1e-8
        counts.append(len(hist))
    assert max(counts) - min(counts) >= 15, counts
    assert min(counts) <= 50 and max(counts) >= 70, counts
