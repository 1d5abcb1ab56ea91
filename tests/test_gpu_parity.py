"""GPU parity: libtdb (sm_100a) vs the reference's golden outputs and the oracle.

Tolerances (BASELINE north star: 1e-10 relative on matrix entries):
  * drop-in pair kernel      <= 1e-13 * max|ref|  (reference twin bound, test_assembly.py:142-161)
  * assembled blocks          <= 1e-11 * max|block| per canonical block, union pattern
  * matvec                    <= 1e-12 relative 2-norm (reference: 1e-13 vs its own dense)
"""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden

pytestmark = pytest.mark.gpu

TOL_BLOCK = 1e-11


@pytest.fixture(scope="module")
def G():
    from paper_1503_07221_b200 import _kernels, assembly, block_system

    return _kernels, assembly, block_system


def test_dropin_regular(G, ico):
    from test_oracle_golden import reg_args

    g = golden("pair_contrib.npz")
    out = G[0].pair_block_contributions(*reg_args(ico, g))
    ref = g["reg_core"]
    assert np.max(np.abs(out - ref)) < 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("case", ["coincident", "edge", "vertex"])
@pytest.mark.parametrize("p", [0, 2])
def test_dropin_singular(G, case, p):
    from test_oracle_golden import sing_args

    g = golden("pair_contrib.npz")
    out = G[0].pair_block_contributions(*sing_args(case, p, g))
    ref = g[f"{case}_p{p}_core"]
    assert np.max(np.abs(out - ref)) < 1e-13 * np.max(np.abs(ref))


def test_dropin_empty_and_shape_errors(G, ico):
    from test_oracle_golden import reg_args

    g = golden("pair_contrib.npz")
    a = list(reg_args(ico, g))
    for k in range(7):
        a[k] = a[k][:0]
    assert G[0].pair_block_contributions(*a).shape == (0, 2, 2, 3, 3)
    b = list(reg_args(ico, g))
    b[2] = b[2][:3]
    with pytest.raises(ValueError):
        G[0].pair_block_contributions(*b)


def test_fixture_block_22(G, two_tri):
    from paper_1503_07221_b200.kernel_weights import tables_for
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    g = TimeGrid(T=2.0, N=3, p=0)
    fx = golden("fixture_block_22.npy")
    A = G[1].assemble_subblocks(two_tri, g, tables_for(g), 2, 2)[0][0].toarray()
    assert np.max(np.abs(A - fx)) < 5e-6
    hi = G[1].assemble_subblocks(two_tri, g, tables_for(g), 2, 2, G[1].QuadratureConfig(8, 8, 8))[0][0]
    hi = hi.toarray()
    assert np.max(np.abs(hi - fx)) < 5e-8
    assert np.max(np.abs(hi - golden("two_tri_22_q888.npy"))) < TOL_BLOCK * np.max(np.abs(hi))


CASES = [
    ("two_tri_N3_p0", 2.0, 3, 0, "two_tri"),
    ("two_tri_N4_p1", 2.0, 4, 1, "two_tri"),
    ("two_tri_N6_p1", 3.0, 6, 1, "two_tri"),
    ("ico_N5_p1", 2.0, 5, 1, "ico"),
    ("sphere80_N6_p1", 2.5, 6, 1, "sphere80"),
    ("ico_N8_p2", 2.0, 8, 2, "ico"),
]


@pytest.mark.parametrize("name,T,N,p,mesh", CASES)
def test_system_blocks_matvec(G, name, T, N, p, mesh, request):
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    m = request.getfixturevalue(mesh)
    g = golden(f"blocks_{name}.npz")
    grid = TimeGrid(T=T, N=N, p=p)
    A = G[2].assemble_system(m, grid)
    positions = [tuple(int(v) for v in r) for r in g["positions"]]
    assert sorted(A.unique_blocks) == positions
    np1 = p + 1
    for kt, it in positions:
        for m2 in range(np1):
            for m1 in range(np1):
                key = f"b_{kt}_{it}_{m2}_{m1}"
                blk = A.unique_blocks[(kt, it)][m2][m1]
                if key not in g.files:
                    assert blk is None
                    continue
                ref = g[key]
                got = blk.toarray()
                scale = np.max(np.abs(ref))
                assert np.max(np.abs(got - ref)) <= TOL_BLOCK * max(scale, 1e-300), (key, scale)
    dense = G[2].reconstruct_dense(A)
    assert np.max(np.abs(dense - g["dense"])) <= TOL_BLOCK * np.max(np.abs(g["dense"]))
    y = A @ g["x7"]
    assert np.linalg.norm(y - g["y7"]) <= 1e-12 * np.linalg.norm(g["y7"])


def test_partial_matvec_and_dimension_check(G, two_tri):
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=2.0, N=4, p=1)
    A = G[2].assemble_system(two_tri, grid)
    m, np1 = two_tri.num_vertices, 2
    x = np.random.default_rng(8).standard_normal(A.shape[1])
    y = A @ x
    lo, hi = 2, 3
    part = A.matvec(x, rows=(lo, hi))
    assert np.allclose(part, y[(lo - 1) * np1 * m : hi * np1 * m], atol=1e-14)
    xz = np.zeros_like(x)
    xz[(lo - 1) * np1 * m : hi * np1 * m] = x[(lo - 1) * np1 * m : hi * np1 * m]
    part = A.matvec(x[(lo - 1) * np1 * m : hi * np1 * m], cols=(lo, hi))
    assert np.allclose(part, A @ xz, atol=1e-14)
    with pytest.raises(ValueError):
        A.matvec(np.zeros(3))


def test_reuse_matches_direct_assembly(G, ico):
    # every logical sub-block of the system equals a from-scratch assembly of that position
    # by the reference (golden direct_*); the reference asserts exact equality against itself
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    g = golden("blocks_ico_N5_p1.npz")
    grid = TimeGrid(T=2.0, N=5, p=1)
    A = G[2].assemble_system(ico, grid)
    for kt in range(1, 6):
        for it in range(1, 6):
            if kt - it <= -2:
                continue
            for m2 in range(2):
                for m1 in range(2):
                    ref = g[f"direct_{kt}_{it}_{m2}_{m1}"]
                    got = A.sub_block(kt, it, m2, m1).toarray()
                    assert np.max(np.abs(got - ref)) <= TOL_BLOCK * max(np.max(np.abs(ref)), 1e-300)


def test_subblock_swap_sign_exact(G, two_tri):
    from paper_1503_07221_b200.kernel_weights import tables_for
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    g = TimeGrid(T=2.0, N=5, p=1)
    S = G[1].assemble_subblocks(two_tri, g, tables_for(g), 3, 3)
    for m1 in range(2):
        for m2 in range(2):
            d = S[m2][m1] - (-1.0) ** (m1 + m2) * S[m1][m2]
            assert (abs(d).max() if d.nnz else 0.0) == 0.0
    Z = G[1].assemble_subblocks(two_tri, g, tables_for(g), 2, 4)
    assert all(s.nnz == 0 for row in Z for s in row)


def test_determinism(G, sphere80):
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=2.5, N=6, p=1)
    A1 = G[2].assemble_system(sphere80, grid)
    A2 = G[2].assemble_system(sphere80, grid)
    for f in range(A1._dev.num_families):
        a = A1._dev.family_arrays(f)
        b = A2._dev.family_arrays(f)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
    x = np.random.default_rng(3).standard_normal(A1.shape[1])
    assert np.array_equal(A1 @ x, A2 @ x)


def test_cfg1_positions_vs_reference(G, cfg1_mesh):
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    g = golden("blocks_cfg1.npz")
    grid = TimeGrid(T=3.9, N=40, p=0)
    A = G[2].assemble_system(cfg1_mesh, grid)
    st = A.stats()
    assert st["units"] == int(g["all_units"].sum())
    assert sorted(A.unique_blocks) == [tuple(int(v) for v in r) for r in g["all_positions"]]
    m = cfg1_mesh.num_vertices
    for (kt, it) in [tuple(int(v) for v in r) for r in g["positions"]]:
        ref = sp.csr_matrix((g[f"b_{kt}_{it}_data"], g[f"b_{kt}_{it}_indices"], g[f"b_{kt}_{it}_indptr"]),
                            shape=(m, m))
        got = A.unique_blocks[(kt, it)][0][0]
        assert got.nnz == ref.nnz, (kt, it)
        assert np.array_equal(got.indptr, ref.indptr) and np.array_equal(got.indices, ref.indices)
        scale = abs(ref).max()
        d = abs(got - ref)
        dmax = d.max() if d.nnz else 0.0
        assert dmax <= 1e-10 * max(scale, 1e-300) or (scale == 0 and dmax < 1e-18), (kt, it, dmax, scale)


def test_distance_bounds_bitwise(G, cfg1_mesh):
    from oracle import assembly as OA

    g = golden("blocks_cfg1.npz")
    tmin, tmax = G[1].tri_distance_bounds(cfg1_mesh, g["bound_rows"])
    assert np.array_equal(tmin, g["tmin_rows"]) and np.array_equal(tmax, g["tmax_rows"])
    from paper_1503_07221_b200.mesh import jittered_cube

    cube = jittered_cube(6, 0.05, 0)
    t1, x1 = OA.tri_distance_bounds(cube)
    t2, x2 = G[1].tri_distance_bounds(cube)
    assert np.array_equal(t1, t2) and np.array_equal(x1, x2)


def test_device_solvers_two_tri(G, two_tri):
    import torch

    from paper_1503_07221_b200.solvers import SolverConfig, dgmres, fgmres, gmres, recursive_preconditioner
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    g = golden("solvers.npz")
    dense = golden("blocks_two_tri_N6_p1.npz")["dense"]
    A = G[2].assemble_system(two_tri, TimeGrid(T=3.0, N=6, p=1))
    b = torch.as_tensor(g["b9"]).cuda()
    xd = np.linalg.solve(dense, g["b9"])
    Av = lambda v: A.matvec(v)
    cfg = SolverConfig(restart=40, tol=1e-12, max_iter=4000, recursion_depth=2, inner_iterations=(2, 6))
    x, hist = fgmres(Av, b, cfg, precond=recursive_preconditioner(A, cfg))
    assert hist[-1] <= 1e-12
    assert np.linalg.norm(x.cpu().numpy() - xd) <= 1e-8 * np.linalg.norm(xd)
    x, hist = gmres(Av, b, SolverConfig(restart=40, tol=1e-12, max_iter=4000))
    assert np.linalg.norm(x.cpu().numpy() - xd) <= 1e-8 * np.linalg.norm(xd)
    x, hist, st = dgmres(Av, b, SolverConfig(restart=20, tol=1e-12, max_iter=4000, deflate_per_restart=2,
                                             max_deflation=8))
    assert np.linalg.norm(x.cpu().numpy() - g["dgm_x"]) <= 1e-8 * np.linalg.norm(g["dgm_x"])
    assert st.rank == int(g["dgm_rank"][0])


def test_device_fgmres_recursive_cfg1_vs_direct(G, cfg1_mesh):
    # config 1 system (E=320, N=40, p=0, L*M = 6480): FGMRES(50, 2(2,10)) at eps=1e-12 vs a
    # dense direct solve of the same assembled matrix (SURVEY 8d solve-parity protocol)
    import torch

    from paper_1503_07221_b200.solvers import SolverConfig, solve
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=3.9, N=40, p=0)
    A = G[2].assemble_system(cfg1_mesh, grid)
    dense = G[2].reconstruct_dense(A)
    b = np.random.default_rng(7).standard_normal(A.shape[0])
    xd = np.linalg.solve(dense, b)
    cfg = SolverConfig(method="fgmres-recursive", restart=50, tol=1e-12, max_iter=2000, recursion_depth=2,
                       inner_iterations=(2, 10))
    x, hist = solve(A, b, cfg)
    assert hist[-1] <= 1e-12
    assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd)


def test_reference_lookalike_inputs(G, two_tri):
    # reference SurfaceMesh / TimeGrid objects (duck-typed) are accepted by the drop-ins
    import types

    g = golden("blocks_two_tri_N4_p1.npz")
    mesh = types.SimpleNamespace(vertices=two_tri.vertices.copy(), triangles=two_tri.triangles.copy())
    grid = types.SimpleNamespace(T=2.0, N=4, p=1)
    A = G[2].assemble_system(mesh, grid)
    assert np.linalg.norm(A @ g["x7"] - g["y7"]) <= 1e-12 * np.linalg.norm(g["y7"])


def test_row_partition_bitwise_and_emulated_allgather(G, cfg1_mesh):
    # every row block's CSR rows and matvec rows are bit-identical to the
    # full system's; the all-gathered x layout is read through the x_map (ranks emulated
    # on one device, the gather is the concatenation an ncclAllGather would produce)
    import torch

    from paper_1503_07221_b200.distributed import DistributedBlockHessenbergMatrix, partition_rows
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=3.9, N=40, p=0)
    A = G[2].assemble_system(cfg1_mesh, grid)
    M = cfg1_mesh.num_vertices
    R = 3
    rows, _ = partition_rows(cfg1_mesh, R)
    parts = [DistributedBlockHessenbergMatrix(cfg1_mesh, grid, rows, r) for r in range(R)]
    assert sum(p.stats()["units_primary"] for p in parts) == A.stats()["units"]
    # CSR rows identical
    for f in range(A._dev.num_families):
        ip, ix, dv = A._dev.family_arrays(f)
        npos = len(A._dev.plan.families[f].positions)
        for r, p in enumerate(parts):
            lip, lix, ldv = p.dev.family_arrays(f)
            for s in range(0, npos, max(1, npos // 5)):
                for k, j in enumerate(rows[r][:: max(1, len(rows[r]) // 7)]):
                    kk = int(np.searchsorted(rows[r], j))
                    a0, a1 = ip[s * M + j], ip[s * M + j + 1]
                    b0, b1 = lip[s * len(rows[r]) + kk], lip[s * len(rows[r]) + kk + 1]
                    assert np.array_equal(ix[a0:a1], lix[b0:b1]) and np.array_equal(dv[a0:a1], ldv[b0:b1])
    x = np.random.default_rng(5).standard_normal(A.shape[1])
    for rws, cls in ((None, None), ((3, 17), (2, 20)), ((21, 40), (1, 40))):
        rlo, rhi = rws or (1, 40)
        clo, chi = cls or (1, 40)
        xs = x[(clo - 1) * M : chi * M]
        y_full = A.matvec(xs, rows=rws, cols=cls)
        ncols = chi - clo + 1
        nmax = max(len(r) for r in rows)
        stacked = torch.zeros((R, ncols, nmax), dtype=torch.float64, device="cuda")
        for r in range(R):
            stacked[r, :, : len(rows[r])] = torch.as_tensor(xs.reshape(ncols, M)[:, rows[r]])
        y = np.zeros(((rhi - rlo + 1), M))
        for r, p in enumerate(parts):
            p._gather = lambda pad, st=stacked: st
            xl = torch.as_tensor(p.local_of(xs, ncols)).cuda()
            yl = p.matvec(xl, rows=rws, cols=cls).cpu().numpy().reshape(rhi - rlo + 1, len(rows[r]))
            y[:, rows[r]] = yl
        # same CSR rows; only the matvec's term grouping (sized per rank) reorders sums
        assert np.linalg.norm(y.ravel() - y_full) <= 1e-14 * np.linalg.norm(y_full)


def test_tiled_matvec_ranges_vs_dense(G, cfg1_mesh):
    # the lag-band tensor-core path (regular lag terms, tdb_band.cu) and the CSR path on
    # the config-1 system, full / half / off-diagonal / quarter / ragged ranges vs dense
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=3.9, N=40, p=0)
    A = G[2].assemble_system(cfg1_mesh, grid)
    dense = G[2].reconstruct_dense(A)
    M = cfg1_mesh.num_vertices
    rng = np.random.default_rng(11)
    kinds = {}
    for rows, cols in [((1, 40), (1, 40)), ((21, 40), (21, 40)), ((21, 40), (1, 20)), ((1, 10), (1, 10)),
                       ((3, 37), (2, 29)), ((11, 20), (1, 10)), ((2, 39), (2, 39)), ((40, 40), (1, 40)),
                       ((1, 40), (5, 5))]:
        x = rng.standard_normal((cols[1] - cols[0] + 1) * M)
        y = A.matvec(x, rows=rows, cols=cols)
        ref = dense[(rows[0] - 1) * M:rows[1] * M, (cols[0] - 1) * M:cols[1] * M] @ x
        assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref), (rows, cols)
        pl = A.matvec_plan(rows, cols)
        kinds[(rows, cols)] = (pl.tiled_terms, pl.csr_terms)
    assert kinds[((1, 40), (1, 40))][0] > 0, kinds       # lag terms on the tensor cores
    assert kinds[((1, 40), (1, 40))][1] > 0, kinds       # boundary terms + the tie lag on CSR


def test_tiled_vs_csr_only_plan_agree(G, cfg1_mesh, tmp_path):
    # the same matvecs with every term on the CSR kernel (TDB_MV_BAND=0, separate
    # process: the switch is read once per process) agree with the default plans
    import os
    import subprocess
    import sys

    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=3.9, N=40, p=0)
    A = G[2].assemble_system(cfg1_mesh, grid)
    M = cfg1_mesh.num_vertices
    x = np.random.default_rng(5).standard_normal(grid.L * M)
    np.save(tmp_path / "x.npy", x)
    ys = [A.matvec(x), A.matvec(x[: 20 * M], rows=(21, 40), cols=(1, 20))]
    assert A.matvec_plan((1, 40), (1, 40)).tiled_terms > 0
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from paper_1503_07221_b200.mesh import icosphere\n"
        "from paper_1503_07221_b200.block_system import assemble_system\n"
        "from paper_1503_07221_b200.temporal_basis import TimeGrid\n"
        "mesh = icosphere(2); g = TimeGrid(T=3.9, N=40, p=0); A = assemble_system(mesh, g)\n"
        "x = np.load(%r); M = mesh.num_vertices\n"
        "assert A.matvec_plan((1, 40), (1, 40)).tiled_terms == 0\n"
        "np.save(%r, np.stack([A.matvec(x), np.pad(A.matvec(x[:20 * M], rows=(21, 40), cols=(1, 20)), (0, 20 * M))]))\n"
    ) % (root, os.path.join(root, "tests"), str(tmp_path / "x.npy"), str(tmp_path / "y.npy"))
    env = dict(os.environ, TDB_MV_BAND="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=root)
    yc = np.load(tmp_path / "y.npy")
    assert np.linalg.norm(ys[0] - yc[0]) <= 1e-13 * np.linalg.norm(yc[0])
    assert np.linalg.norm(ys[1] - yc[1][: 20 * M]) <= 1e-13 * np.linalg.norm(yc[1][: 20 * M])
    # these 40-row plans run on k_band_direct (<= 6 time tiles); TDB_BAND_DIRECT=0 puts them
    # on the shared-memory ring kernel k_band_mv: same records, same DMMA order per part
    code2 = code.replace("tiled_terms == 0", "tiled_terms > 0")
    subprocess.run([sys.executable, "-c", code2], check=True, env=dict(os.environ, TDB_BAND_DIRECT="0"), cwd=root)
    yr = np.load(tmp_path / "y.npy")
    assert np.linalg.norm(ys[0] - yr[0]) <= 1e-13 * np.linalg.norm(yr[0])
    assert np.linalg.norm(ys[1] - yr[1][: 20 * M]) <= 1e-13 * np.linalg.norm(yr[1][: 20 * M])


def test_matvec_long_time_axis_row_chunks(G, ico):
    # N > 384 block rows: the matvec is applied in row chunks of MAX_PLAN_ROWS, one plan each
    # (ADVICE r01); compared with the oracle's reference-order block matvec
    from oracle import assembly as OA
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=10.0, N=401, p=0)
    A = G[2].assemble_system(ico, grid)
    x = np.random.default_rng(4).standard_normal(A.shape[1])
    y = A.matvec(x)
    y_ref = OA.matvec(grid, ico.num_vertices, ico.diameter, A.unique_blocks, x)
    assert np.linalg.norm(y - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
    A.MAX_PLAN_ROWS = 7  # many chunks, ragged last one
    y7 = A.matvec(x, rows=(3, 390), cols=(1, 401))
    assert np.linalg.norm(y7 - y_ref[2 * ico.num_vertices:390 * ico.num_vertices]) <= 1e-12 * np.linalg.norm(y7)


def test_position_batches_bitwise(G, cfg1_mesh, monkeypatch):
    # a capped partial buffer (TDB_PARTIAL_GB) splits every family's positions into lag
    # batches (plan -> counts per batch, scan, then plan -> quadrature -> fill per batch);
    # the assembled system must be bit-identical to the one-batch assembly
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=3.9, N=40, p=0)
    A1 = G[2].assemble_system(cfg1_mesh, grid)
    monkeypatch.setenv("TDB_PARTIAL_GB", "0.03")
    A2 = G[2].assemble_system(cfg1_mesh, grid)
    monkeypatch.delenv("TDB_PARTIAL_GB")
    assert A2._dev.num_families == A1._dev.num_families
    for f in range(A1._dev.num_families):
        for u, v in zip(A1._dev.family_arrays(f), A2._dev.family_arrays(f)):
            assert np.array_equal(u, v)
    s1, s2 = A1.stats(), A2.stats()
    assert s1["units"] == s2["units"] and s1["n_in"] == s2["n_in"]
    assert A1._dev.position_units() == A2._dev.position_units()
    A2._dev.rerun()  # re-run from the resident inputs, still identical
    for f in range(A1._dev.num_families):
        assert np.array_equal(A1._dev.family_arrays(f)[2], A2._dev.family_arrays(f)[2])


def test_cell_owner_kernel_matches_k_quad(G, cfg1_mesh, monkeypatch):
    # the regular pairs of the dt-grid families run on k_quad_cells (csrc/tdb_quad_cells.cuh),
    # the singular cases and the singleton families on k_quad; TDB_CELLS=0 (read at system
    # creation) keeps everything on k_quad.  Same rule points, tables and arithmetic per
    # evaluation, different summation order: the blocks agree to roundoff.
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=3.9, N=40, p=0)
    A1 = G[2].assemble_system(cfg1_mesh, grid)
    monkeypatch.setenv("TDB_CELLS", "0")
    A0 = G[2].assemble_system(cfg1_mesh, grid)
    monkeypatch.delenv("TDB_CELLS")
    s1, s0 = A1.stats(), A0.stats()
    assert s1["pairs_cells"] > 0 and s1["n_in_cells"] > 0 and s1["ms_quad_cells"] > 0.0
    assert s0["pairs_cells"] == 0 and s0["n_in_cells"] == 0
    # every in-support (unit, point) evaluation is done exactly once by one of the kernels
    assert s1["units"] == s0["units"] and s1["n_in"] == s0["n_in"]
    assert 0 < s1["items"] < s0["items"]  # no k_quad work item for a fully covered regular pair
    assert A1._dev.position_units() == A0._dev.position_units()
    for f in range(A1._dev.num_families):
        p1, i1, d1 = A1._dev.family_arrays(f)
        p0, i0, d0 = A0._dev.family_arrays(f)
        assert np.array_equal(p1, p0) and np.array_equal(i1, i0)
        assert np.all(np.isfinite(d1))
        assert np.abs(d1 - d0).max() <= 1e-13 * np.abs(d0).max()
    # p = 1 tables are off the kernel's grid: everything stays on k_quad
    A2 = G[2].assemble_system(cfg1_mesh, TimeGrid(T=1.0, N=5, p=1))
    assert A2.stats()["pairs_cells"] == 0


def test_lag_subsets_bitwise_equal_full_system(G, cfg1_mesh):
    # a system that holds only a lag range of every family (lag-sharded ranks, position
    # batches) must produce the same bits as the full system, whatever the range: the
    # pair windows are clipped at the range ends, families may shrink to one position
    # (kernel selection and the k_quad_cells summation order must not depend on either)
    from paper_1503_07221_b200 import _lib
    from paper_1503_07221_b200.assembly import DeviceAssembly, build_plan
    from paper_1503_07221_b200.block_system import canonical_positions
    from paper_1503_07221_b200.distributed import partition_lags
    from paper_1503_07221_b200.kernel_weights import tables_for
    from paper_1503_07221_b200.temporal_basis import TimeGrid

    grid = TimeGrid(T=3.9, N=40, p=0)
    tables = tables_for(grid)
    pos = canonical_positions(grid, cfg1_mesh.diameter)
    ctx = _lib.default_context(None)
    full = DeviceAssembly(cfg1_mesh, build_plan(cfg1_mesh, grid, tables, pos), ctx)
    ref = {p: full.position_blocks(*p)[0][0] for p in full.plan.where}
    seen = set()
    for groups, picks in ((2, (0, 1)), (5, (1, 4)), (24, (0, 7, 23))):
        parts = partition_lags(grid, pos, groups)
        for lg in picks:
            if not parts[lg]:
                continue
            d = DeviceAssembly(cfg1_mesh, build_plan(cfg1_mesh, grid, tables, parts[lg]), ctx)
            for p in d.plan.where:
                a, b = d.position_blocks(*p)[0][0], ref[p]
                assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices), (groups, lg, p)
                assert np.array_equal(a.data, b.data), (groups, lg, p)
                seen.add(p)
    assert len(seen) > len(ref) // 2
