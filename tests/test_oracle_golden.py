"""Pin the oracle (oracle/) against the reference's own outputs before trusting it.

Golden vectors from tests/golden/make_golden.py (the reference package run in
this container): compiled _core outputs, assembled canonical blocks, matvecs,
and the reference test suite's FIXTURE_BLOCK_22 known answer.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import assembly as OA
from paper_1503_07221_b200.assembly import PsiPack, QuadratureConfig
from paper_1503_07221_b200.kernel_weights import tables_for
from paper_1503_07221_b200.mesh import icosphere
from paper_1503_07221_b200.quadrature import pair_rule_regular, singular_rule
from paper_1503_07221_b200.temporal_basis import TimeGrid


def reg_args(ico, g):
    pack = PsiPack.build(tables_for(TimeGrid(T=6.0, N=10, p=1)), TimeGrid(T=6.0, N=10, p=1), 4, 2)
    ex, ey = g["reg_ex"], g["reg_ey"]
    xh, yh, wq = pair_rule_regular(4)
    return (ico.corners[ex], ico.corners[ey], 2.0 * ico.areas[ex], 2.0 * ico.areas[ey],
            np.einsum("pd,pd->p", ico.normals[ex], ico.normals[ey]), ico.curls[ey], ico.curls[ex],
            xh, yh, wq, pack)


def sing_args(case, p, g):
    m1 = icosphere(1)
    grid = TimeGrid(T=2.0, N=5, p=p)
    pk = PsiPack.build(tables_for(grid), grid, 2, 2)
    parr, lx, ly = g[f"{case}_p{p}_pairs"], g[f"{case}_p{p}_lx"], g[f"{case}_p{p}_ly"]
    ax = np.arange(len(parr))
    return (m1.corners[parr[:, 0]][ax[:, None], lx], m1.corners[parr[:, 1]][ax[:, None], ly],
            2.0 * m1.areas[parr[:, 0]], 2.0 * m1.areas[parr[:, 1]],
            np.einsum("pd,pd->p", m1.normals[parr[:, 0]], m1.normals[parr[:, 1]]),
            m1.curls[parr[:, 1]][ax[:, None], ly], m1.curls[parr[:, 0]][ax[:, None], lx],
            *singular_rule(case, 5, 2, 2), pk)


def test_c_kernel_matches_compiled_reference_regular(ico):
    g = golden("pair_contrib.npz")
    out = OA.c_pair_block_contributions(*reg_args(ico, g))
    ref = g["reg_core"]
    assert np.max(np.abs(out - ref)) <= 1e-14 * np.max(np.abs(ref))
    # the reference's own twin agreement bound (test_assembly.py:142-161)
    assert np.max(np.abs(out - g["reg_fallback"])) < 1e-13 * np.max(np.abs(g["reg_fallback"]))


@pytest.mark.parametrize("case", ["coincident", "edge", "vertex"])
@pytest.mark.parametrize("p", [0, 2])
def test_c_kernel_matches_compiled_reference_singular(case, p):
    g = golden("pair_contrib.npz")
    out = OA.c_pair_block_contributions(*sing_args(case, p, g))
    ref = g[f"{case}_p{p}_core"]
    assert np.max(np.abs(out - ref)) <= 1e-14 * np.max(np.abs(ref))


def test_ref_core_build_matches_golden(ico):
    core = OA.ref_core()
    if core is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    g = golden("pair_contrib.npz")
    assert np.array_equal(core.pair_block_contributions(*reg_args(ico, g)), g["reg_core"])


def test_fixture_block_22(two_tri):
    fx = golden("fixture_block_22.npy")
    g = TimeGrid(T=2.0, N=3, p=0)
    asm = OA.OracleAssembler(two_tri, g, tables_for(g))
    A = asm.subblocks(2, 2)[0][0].toarray()
    assert np.max(np.abs(A - fx)) < 5e-6
    hi = OA.OracleAssembler(two_tri, g, tables_for(g), QuadratureConfig(8, 8, 8)).subblocks(2, 2)[0][0].toarray()
    assert np.max(np.abs(hi - fx)) < 5e-8
    assert np.max(np.abs(hi - golden("two_tri_22_q888.npy"))) <= 1e-13 * np.max(np.abs(hi))


@pytest.mark.parametrize("name,T,N,p,mesh", [
    ("two_tri_N3_p0", 2.0, 3, 0, "two_tri"),
    ("two_tri_N4_p1", 2.0, 4, 1, "two_tri"),
    ("ico_N5_p1", 2.0, 5, 1, "ico"),
])
def test_oracle_blocks_and_matvec(name, T, N, p, mesh, request):
    m = request.getfixturevalue(mesh)
    g = golden(f"blocks_{name}.npz")
    grid = TimeGrid(T=T, N=N, p=p)
    asm = OA.OracleAssembler(m, grid, tables_for(grid))
    positions = [tuple(int(v) for v in r) for r in g["positions"]]
    blocks = OA.canonical_blocks(asm, positions)
    np1 = p + 1
    for kt, it in positions:
        for m2 in range(np1):
            for m1 in range(np1):
                key = f"b_{kt}_{it}_{m2}_{m1}"
                if key in g.files:
                    ref = g[key]
                    got = blocks[(kt, it)][m2][m1].toarray()
                    assert np.max(np.abs(got - ref)) <= 1e-13 * max(1e-300, np.max(np.abs(ref))), key
    y = OA.matvec(grid, m.num_vertices, m.diameter, blocks, g["x7"])
    assert np.linalg.norm(y - g["y7"]) <= 1e-13 * np.linalg.norm(g["y7"])
    assert np.linalg.norm(g["dense"] @ g["x7"] - g["y7"]) <= 1e-13 * np.linalg.norm(g["y7"])


def test_oracle_bounds_and_units_cfg1(cfg1_mesh):
    g = golden("blocks_cfg1.npz")
    rows = g["bound_rows"]
    tmin, tmax = OA.tri_distance_bounds(cfg1_mesh, rows)
    assert np.array_equal(tmin, g["tmin_rows"]) and np.array_equal(tmax, g["tmax_rows"])


def test_oracle_cfg1_regular_positions(cfg1_mesh):
    # cheap (regular-dominated) config-1 positions; the full set runs in the GPU parity tests
    g = golden("blocks_cfg1.npz")
    grid = TimeGrid(T=3.9, N=40, p=0)
    asm = OA.OracleAssembler(cfg1_mesh, grid, tables_for(grid))
    for kt, it in ((24, 2), (40, 20)):
        got = asm.subblocks(kt, it)[0][0]
        ref_shape = (cfg1_mesh.num_vertices,) * 2
        import scipy.sparse as sp

        ref = sp.csr_matrix((g[f"b_{kt}_{it}_data"], g[f"b_{kt}_{it}_indices"], g[f"b_{kt}_{it}_indptr"]),
                            shape=ref_shape)
        d = abs(got - ref)
        scale = max(abs(ref).max(), 1e-300)
        assert (d.max() if d.nnz else 0.0) <= 1e-13 * scale
        assert got.nnz == ref.nnz
