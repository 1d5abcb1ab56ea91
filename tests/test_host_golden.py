"""Host-side inputs of the hot path are bit-identical to the reference's.

Golden vectors: tests/golden/{rules,meshes,tables_*}.npz, made by
tests/golden/make_golden.py from the reference package itself.
"""

import numpy as np
import pytest

from conftest import golden
from paper_1503_07221_b200 import kernel_weights as K
from paper_1503_07221_b200 import mesh as M
from paper_1503_07221_b200 import quadrature as Q
from paper_1503_07221_b200.temporal_basis import TimeGrid


def test_triangle_and_regular_rules_bitwise():
    g = golden("rules.npz")
    for q in (3, 4):
        p, w = Q.triangle_rule(q)
        assert np.array_equal(p, g[f"tri{q}_pts"]) and np.array_equal(w, g[f"tri{q}_w"])
    x, y, w = Q.pair_rule_regular(4)
    assert np.array_equal(x, g["reg4_x"]) and np.array_equal(y, g["reg4_y"]) and np.array_equal(w, g["reg4_w"])
    assert w.sum() == pytest.approx(0.25, abs=1e-14)


@pytest.mark.parametrize("case", ["coincident", "edge", "vertex"])
def test_singular_rules_bitwise(case):
    g = golden("rules.npz")
    x, y, w = Q.singular_rule(case, 5, 1, 1)
    assert np.array_equal(x, g[f"{case}_1_x"]) and np.array_equal(y, g[f"{case}_1_y"])
    assert np.array_equal(w, g[f"{case}_1_w"])
    x, y, w = Q.singular_rule(case, 5, 8, 2)
    assert len(w) == int(g[f"{case}_8_n"][0])
    idx = g[f"{case}_8_idx"]
    assert np.array_equal(np.column_stack([x[idx], y[idx], w[idx]]), g[f"{case}_8_rows"])
    mom = np.array([w.sum(), (w * x[:, 0]).sum(), (w * x[:, 1]).sum(), (w * y[:, 0]).sum(),
                    (w * y[:, 1]).sum(), (w * np.linalg.norm(x - y, axis=1)).sum()])
    assert np.array_equal(mom, g[f"{case}_8_mom"])
    assert w.sum() == pytest.approx(0.25, abs=1e-13)


def test_coincident_known_integral():
    # reference known answer: int_T int_T 1/(4 pi |x-y|) = 0.079821446904 (test_quadrature.py:78-95)
    xh, yh, wq = Q.singular_rule("coincident", 5, 4, 2)
    val = np.sum(wq / (4.0 * np.pi * np.linalg.norm(xh - yh, axis=1)))
    assert val == pytest.approx(0.079821446904, abs=1e-8)


def test_meshes_bitwise():
    g = golden("meshes.npz")
    for lv in range(4):
        m = M.icosphere(lv)
        assert np.array_equal(m.vertices, g[f"ico{lv}_v"]) and np.array_equal(m.triangles, g[f"ico{lv}_t"])
        if lv:
            assert m.diameter == float(g[f"ico{lv}_diam"][0])
    for name, lv in (("sphere80", 1), ("sphere320", 2)):
        m = M.icosphere(lv)
        scale = np.sqrt(4.0 * np.pi / m.areas.sum())
        assert np.array_equal(m.vertices * scale, g[f"{name}_v"])
        assert np.array_equal(m.triangles, g[f"{name}_t"])


def test_cube_generator_valid():
    c = M.jittered_cube(16, 0.05, 0)
    assert c.num_triangles == 3072 and c.num_vertices == 1538
    c.validate_closed()
    assert c.signed_volume > 0
    assert 1.70 < c.diameter < 1.76


@pytest.mark.parametrize("T,N,p", [(2.0, 3, 0), (2.0, 4, 1), (2.0, 5, 2), (3.9, 40, 0), (3.0, 6, 1)])
def test_tables_match_reference(T, N, p):
    g = golden(f"tables_T{T}_N{N}_p{p}.npz")
    tabs = K.build_tables(TimeGrid(T=T, N=N, p=p))
    seen = 0
    for key, tbl in tabs.tables.items():
        tilde, ki, kk, m1, m2 = key
        name = f"{int(tilde)}_{ki}_{kk}_{m1}_{m2}"
        if tbl is None:
            assert name + "_none" in g.files
            continue
        assert np.array_equal(np.array([tbl.lo, tbl.hi]), g[name + "_dom"])
        ref = g[name]
        assert np.max(np.abs(tbl.coeffs - ref)) <= 1e-14 * max(1.0, np.max(np.abs(ref)))
        seen += 1
    assert seen > 0


def test_oracle_rhs_matches_reference(two_tri):
    # the oracle's host restatement of the reference loop (the product's RHS is GPU-only,
    # tests/test_gpu_rhs.py); the Gaussian datum's host callback is the product's
    from oracle.assembly import assemble_rhs
    from paper_1503_07221_b200.assembly import gaussian_pulse_neumann

    g = golden("rhs.npz")
    m = M.icosphere(2)
    b = assemble_rhs(m, TimeGrid(T=3.9, N=40, p=0), gaussian_pulse_neumann(m))
    assert np.max(np.abs(b - g["cfg1_pulse"])) <= 1e-14 * np.max(np.abs(g["cfg1_pulse"]))

    def gs(X, t):
        return (X[:, 0] + 2 * X[:, 1] - X[:, 2]) * np.sin(3 * t) * t * t * np.exp(-t)

    b2 = assemble_rhs(two_tri, TimeGrid(T=3.0, N=5, p=1), gs)
    assert np.max(np.abs(b2 - g["two_tri_smooth"])) <= 1e-14 * np.max(np.abs(g["two_tri_smooth"]))


def test_touching_pairs_vectorised_matches_loop():
    from paper_1503_07221_b200.mesh import _touching_pairs_loop, icosphere, jittered_cube, touching_pairs

    for m in (icosphere(2), jittered_cube(4, 0.05, 1)):
        a, b = touching_pairs(m), _touching_pairs_loop(m)
        for case in ("coincident", "edge", "vertex"):
            for x, y in zip(a[case], b[case]):
                assert np.array_equal(x, y)
