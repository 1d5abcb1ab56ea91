"""Row-block sharding host logic on CPU with world_size 2 (gloo): partition,
all-gather layout / x_map, and the distributed Krylov solvers."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1503_07221_b200.distributed import gathered_x_map, partition_rows
from paper_1503_07221_b200.mesh import icosphere


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("nparts", [1, 2, 3, 8])
def test_partition_rows_cover_and_halo(nparts):
    mesh = icosphere(3)
    rows, tests = partition_rows(mesh, nparts)
    allrows = np.concatenate(rows)
    assert np.array_equal(np.sort(allrows), np.arange(mesh.num_vertices))
    off, ids = mesh.star_csr
    for r in range(nparts):
        for j in rows[r][:50]:
            assert set(ids[off[j] : off[j + 1]]) <= set(tests[r])
    # halo: duplicated test triangles stay a small fraction (spatially compact blocks)
    dup = sum(len(t) for t in tests) / mesh.num_triangles
    assert dup <= 1.0 + 0.12 * (nparts - 1)
    sizes = [len(r) for r in rows]
    assert max(sizes) <= 1.25 * (mesh.num_vertices / nparts) + 8


def test_gathered_x_map_roundtrip():
    mesh = icosphere(2)
    rows, _ = partition_rows(mesh, 3)
    M, ncols = mesh.num_vertices, 5
    nmax = max(len(r) for r in rows)
    x = np.random.default_rng(0).standard_normal((ncols, M))
    gathered = np.zeros((3, ncols, nmax))
    for r in range(3):
        gathered[r, :, : len(rows[r])] = x[:, rows[r]]
    xmap = gathered_x_map(rows, M, ncols, nmax)
    flat = gathered.ravel()
    for c in range(ncols):
        assert np.array_equal(flat[xmap + c * nmax], x[c])


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1503_07221_b200 import solvers as S

    rng = np.random.default_rng(3)
    ncols, M = 6, 40
    n = ncols * M
    D = np.eye(n) + (0.4 / np.sqrt(n)) * rng.standard_normal((n, n))
    b = rng.standard_normal(n)
    rows = [np.arange(0, 17), np.arange(17, 40)]  # vertex rows per rank
    mine = rows[rank]
    idx = (np.arange(ncols)[:, None] * M + mine[None, :]).ravel()  # global entries of local piece
    Dl = torch.as_tensor(D[idx])  # local rows of the operator

    nmax = max(len(r) for r in rows)

    def apply_A(x_local):
        # same padded rank-major all-gather as DistributedBlockHessenbergMatrix
        pad = torch.zeros((ncols, nmax), dtype=torch.float64)
        pad[:, : len(mine)] = x_local.view(ncols, len(mine))
        pieces = [torch.zeros((ncols, nmax), dtype=torch.float64) for _ in rows]
        dist.all_gather(pieces, pad)
        full = torch.zeros(n, dtype=torch.float64)
        for r, p in zip(rows, pieces):
            ridx = (np.arange(ncols)[:, None] * M + r[None, :]).ravel()
            full[torch.as_tensor(ridx)] = p[:, : len(r)].reshape(-1)
        return Dl @ full

    S.set_comm(S.TorchDistComm())
    cfg = S.SolverConfig(restart=20, tol=1e-12, max_iter=500)
    x, hist = S.gmres(apply_A, torch.as_tensor(b[idx]), cfg)
    xd, histd, st = S.dgmres(apply_A, torch.as_tensor(b[idx]), S.SolverConfig(restart=15, tol=1e-12, max_iter=600,
                                                                             deflate_per_restart=2, max_deflation=6))
    S.set_comm(None)
    out[rank] = (idx, x.numpy(), len(hist), xd.numpy(), st.rank)
    dist.destroy_process_group()


def test_distributed_krylov_matches_single_process():
    # spawn-context manager: a forked manager process leaves the parent's BLAS
    # thread pool deadlocked for later tests
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    port = free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    out = dict(out)
    mgr.shutdown()
    rng = np.random.default_rng(3)
    n = 240
    D = np.eye(n) + (0.4 / np.sqrt(n)) * rng.standard_normal((n, n))
    b = rng.standard_normal(n)
    x = np.zeros(n)
    xd = np.zeros(n)
    for r in range(2):
        idx, xr, nit, xdr, rk = out[r]
        x[idx] = xr
        xd[idx] = xdr
    ref = np.linalg.solve(D, b)
    assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)
    assert np.linalg.norm(xd - ref) <= 1e-10 * np.linalg.norm(ref)
    assert out[0][2] == out[1][2]  # replicated Hessenberg logic: same iteration count on all ranks
    assert out[0][4] == out[1][4]


@pytest.mark.parametrize("groups", [1, 2, 3, 4])
def test_partition_lags_contiguous_cover(groups):
    from paper_1503_07221_b200.block_system import canonical_positions
    from paper_1503_07221_b200.configs import get_config
    from paper_1503_07221_b200.distributed import partition_lags
    from paper_1503_07221_b200.temporal_basis import timestep_kind

    cfg = get_config(2)
    mesh, grid = cfg.mesh(), cfg.grid()
    pos = canonical_positions(grid, mesh.diameter)
    parts = partition_lags(grid, pos, groups)
    flat = [p for part in parts for p in part]
    assert sorted(flat) == sorted(pos) and len(flat) == len(set(flat))
    for part in parts:  # every family's share is a run of consecutive lags
        fam = {}
        for kt, it in part:
            fam.setdefault((timestep_kind(grid, it), timestep_kind(grid, kt)), []).append(kt - it)
        for lags in fam.values():
            lags.sort()
            assert lags == list(range(lags[0], lags[0] + len(lags)))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 8  # <= 1 per family (up to 7 families)
