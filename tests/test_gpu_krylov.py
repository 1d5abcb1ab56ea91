"""GPU tests of the device-side Krylov pieces (csrc/tdb_krylov.cu) and of the
caching device allocator (tdb_context.cu).

* tdb_krylov_arnoldi: one fused step (two classical Gram-Schmidt passes, norm,
  Givens update of the reference's _gmres_cycle_raw, solvers.py:189-215,
  normalisation) against a float64 numpy restatement, on cluster sizes 1..16.
* repeated assemble / destroy cycles reuse cached device blocks and reproduce
  the blocks bit for bit.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _np_step(V, w, k, H, cs, sn, g, st):
    h = np.zeros(k + 1)
    for _ in range(2):
        c = V[: k + 1] @ w
        w = w - V[: k + 1].T @ c
        h += c
    hk = np.linalg.norm(w)
    col = np.concatenate([h, [hk]])
    H[: k + 2, k] = col
    for j in range(k):
        t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
        H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
        H[j, k] = t
    d = np.hypot(H[k, k], H[k + 1, k])
    cs[k], sn[k] = H[k, k] / d, H[k + 1, k] / d
    H[k, k] = d
    g[k + 1] = -sn[k] * g[k]
    g[k] = cs[k] * g[k]
    H[k + 1, k] = 0.0
    return col, w / hk


@pytest.mark.parametrize("n", [100, 5000, 40000])
def test_fused_arnoldi_matches_numpy(n):
    import torch

    from paper_1503_07221_b200 import _lib

    rng = np.random.default_rng(n)
    m = 12
    L = _lib.LIB
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    b = rng.standard_normal(n)
    V = np.zeros((m, n))
    V[0] = b / np.linalg.norm(b)
    Hn = np.zeros((m + 1, m))
    csn, snn, gn = np.zeros(m), np.zeros(m), np.zeros(m + 1)
    gn[0] = np.linalg.norm(b)
    Vd = torch.as_tensor(V).cuda()
    Hd = torch.zeros((m + 1, m), dtype=torch.float64, device="cuda")
    csd = torch.zeros(m, dtype=torch.float64, device="cuda")
    snd = torch.zeros(m, dtype=torch.float64, device="cuda")
    gd = torch.zeros(m + 1, dtype=torch.float64, device="cuda")
    st = torch.zeros(_lib.KS_NSTATE, dtype=torch.float64, device="cuda")
    hcol = torch.zeros(m + 1, dtype=torch.float64, device="cuda")
    beta = torch.tensor([np.linalg.norm(b)], dtype=torch.float64, device="cuda")
    _lib.check(L.tdb_krylov_init(p(st), p(beta), 1e-14, p(gd), stream))
    A = rng.standard_normal((n, n)) / np.sqrt(n) if n <= 5000 else None
    for k in range(m - 1):
        z = V[k]
        w = A @ z if A is not None else np.roll(z, 1) * (1.0 + 0.01 * k) + 0.1 * z
        wd = torch.as_tensor(w).cuda()
        _lib.check(L.tdb_krylov_arnoldi(p(Vd), n, n, k, p(wd), p(hcol), p(st), p(Hd), m, p(csd), p(snd), p(gd),
                                        p(Vd[k + 1]), stream))
        col, V[k + 1] = _np_step(V, w, k, Hn, csn, snn, gn, None)
        torch.cuda.synchronize()
        got = hcol[: k + 2].cpu().numpy()
        assert np.allclose(got, col, rtol=1e-12, atol=1e-13 * np.abs(col).max()), (k, got, col)
        assert np.allclose(Vd[k + 1].cpu().numpy(), V[k + 1], rtol=1e-10, atol=1e-12)
        Vd[k + 1].copy_(torch.as_tensor(V[k + 1]))  # follow the numpy basis exactly
    assert np.allclose(gd.cpu().numpy(), gn, rtol=1e-10, atol=1e-12 * abs(gn[0]))
    assert np.allclose(Hd.cpu().numpy(), Hn, rtol=1e-10, atol=1e-12)
    assert int(st[_lib.KS_KDONE].item()) == m - 1


def test_repeated_assembly_reuses_memory_bitwise():
    from paper_1503_07221_b200 import _lib
    from paper_1503_07221_b200.block_system import assemble_system
    from paper_1503_07221_b200.mesh import icosphere
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    mesh, grid = icosphere(2), TimeGrid(T=3.9, N=40, p=0)
    ref = None
    for it in range(3):
        A = assemble_system(mesh, grid)
        arrays = [A._dev.family_arrays(f) for f in range(A._dev.num_families)]
        if ref is None:
            ref = [tuple(np.array(a) for a in fam) for fam in arrays]
        else:
            for (i0, x0, d0), (i1, x1, d1) in zip(ref, arrays):
                assert np.array_equal(i0, i1) and np.array_equal(x0, x1) and np.array_equal(d0, d1)
        del A
    _lib.check(_lib.LIB.tdb_release_cached_memory())
