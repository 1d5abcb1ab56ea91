"""Generate the golden fixtures in tests/golden/ from the REFERENCE package itself.

Run in the build container only (needs /root/reference; never on the GPU box):

    python tests/golden/make_golden.py [--refpkg /tmp/refpkg]

It copies /root/reference/pkg to a scratch dir (read-only source), builds the
reference's Cython kernel there, imports ``tdbem`` and records:

  rules.npz         reference quadrature rules (quadrature.py) - full arrays for
                    small rules, moments + sampled rows for the n_rad=8 ones
  meshes.npz        icosahedron / refinements / area-scaled sphere80, sphere320
                    (the reference's mesh fixtures, read with its load_mesh)
  tables_*.npz      PrototypeTables coefficients for the grids the tests use
  pair_contrib.npz  _core (compiled) and _fallback outputs of
                    pair_block_contributions on regular and singular pair groups
  blocks_*.npz      assembled canonical blocks (assemble_system /
                    assemble_subblocks), dense reconstructions and matvecs
  fixture_block_22.npy  the reference test suite's FIXTURE_BLOCK_22
                    (tests/test_assembly.py:27-35), read from the test module
"""

from __future__ import annotations

import argparse
import importlib.util
import os
import shutil
import subprocess
import sys

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))


def prepare(refpkg: str):
    if not os.path.isdir(os.path.join(refpkg, "src", "tdbem")):
        shutil.copytree("/root/reference/pkg", refpkg)
    so = [f for f in os.listdir(os.path.join(refpkg, "src", "tdbem", "_kernels")) if f.endswith(".so")]
    if not so:
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=refpkg, check=True,
                       capture_output=True)
    sys.path.insert(0, os.path.join(refpkg, "src"))


def csr_pack(prefix, m, out):
    m = m.tocsr()
    m.sort_indices()
    out[prefix + "_indptr"] = m.indptr.astype(np.int64)
    out[prefix + "_indices"] = m.indices.astype(np.int32)
    out[prefix + "_data"] = m.data


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--refpkg", default="/tmp/refpkg")
    ap.add_argument("--skip-cfg1", action="store_true")
    args = ap.parse_args()
    prepare(args.refpkg)

    import tdbem._kernels as K
    from tdbem._kernels import _core, _fallback
    from tdbem.assembly import PsiPack, QuadratureConfig, assemble_subblocks, block_pattern
    from tdbem.block_system import assemble_system, canonical_position, reconstruct_dense
    from tdbem.kernel_weights import build_tables, tables_for
    from tdbem.mesh import SurfaceMesh, icosahedron, load_mesh, refine
    from tdbem.quadrature import pair_rule_regular, singular_rule, triangle_rule
    from tdbem.temporal_basis import TimeGrid

    assert K.backend_name == "compiled", K.backend_name

    # ---- FIXTURE_BLOCK_22 straight from the reference test module ----
    spec = importlib.util.spec_from_file_location(
        "ref_test_assembly", os.path.join(args.refpkg, "tests", "test_assembly.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.path.insert(0, os.path.join(args.refpkg, "tests"))
    spec.loader.exec_module(mod)
    np.save(os.path.join(OUT, "fixture_block_22.npy"), np.asarray(mod.FIXTURE_BLOCK_22))

    # ---- rules ----
    r = {}
    for q in (3, 4):
        p, w = triangle_rule(q)
        r[f"tri{q}_pts"], r[f"tri{q}_w"] = p, w
    xh, yh, w = pair_rule_regular(4)
    r["reg4_x"], r["reg4_y"], r["reg4_w"] = xh, yh, w
    for case in ("coincident", "edge", "vertex"):
        xh, yh, w = singular_rule(case, 5, 1, 1)
        r[f"{case}_1_x"], r[f"{case}_1_y"], r[f"{case}_1_w"] = xh, yh, w
        xh, yh, w = singular_rule(case, 5, 8, 2)
        idx = np.linspace(0, len(w) - 1, 64).astype(np.int64)
        r[f"{case}_8_n"] = np.array([len(w)])
        r[f"{case}_8_idx"] = idx
        r[f"{case}_8_rows"] = np.column_stack([xh[idx], yh[idx], w[idx]])
        r[f"{case}_8_mom"] = np.array([w.sum(), (w * xh[:, 0]).sum(), (w * xh[:, 1]).sum(),
                                       (w * yh[:, 0]).sum(), (w * yh[:, 1]).sum(),
                                       (w * np.linalg.norm(xh - yh, axis=1)).sum()])
    np.savez_compressed(os.path.join(OUT, "rules.npz"), **r)

    # ---- meshes ----
    mm = {}
    ico = icosahedron()
    m = ico
    for lv in range(1, 4):
        m = refine(m, project_unit_sphere=True)
        mm[f"ico{lv}_v"], mm[f"ico{lv}_t"] = m.vertices, m.triangles
        mm[f"ico{lv}_diam"] = np.array([m.diameter])
    mm["ico0_v"], mm["ico0_t"] = ico.vertices, ico.triangles
    for name in ("sphere80", "sphere320"):
        s = load_mesh(os.path.join(args.refpkg, "meshes", f"{name}.off"))
        mm[f"{name}_v"], mm[f"{name}_t"] = s.vertices, s.triangles
    np.savez_compressed(os.path.join(OUT, "meshes.npz"), **mm)

    # ---- tables ----
    for (T, N, p) in ((2.0, 3, 0), (2.0, 4, 1), (2.0, 5, 2), (3.9, 40, 0), (3.0, 6, 1)):
        g = TimeGrid(T=T, N=N, p=p)
        tabs = build_tables(g)
        tt = {}
        for key, tbl in tabs.tables.items():
            tilde, ki, kk, m1, m2 = key
            name = f"{int(tilde)}_{ki}_{kk}_{m1}_{m2}"
            if tbl is None:
                tt[name + "_none"] = np.array([1])
            else:
                tt[name] = tbl.coeffs
                tt[name + "_dom"] = np.array([tbl.lo, tbl.hi])
        np.savez_compressed(os.path.join(OUT, f"tables_T{T}_N{N}_p{p}.npz"), **tt)

    # ---- pair_block_contributions: regular (test_core_matches_fallback setup) ----
    pc = {}
    g = TimeGrid(T=6.0, N=10, p=1)
    pack = PsiPack.build(tables_for(g), g, 4, 2)
    rng = np.random.default_rng(0)
    n = 64
    ex = rng.integers(0, ico.num_triangles, n)
    ey = (ex + 1 + rng.integers(0, ico.num_triangles - 1, n)) % ico.num_triangles
    xh, yh, wq = pair_rule_regular(4)
    a = (ico.corners[ex], ico.corners[ey], 2.0 * ico.areas[ex], 2.0 * ico.areas[ey],
         np.einsum("pd,pd->p", ico.normals[ex], ico.normals[ey]), ico.curls[ey], ico.curls[ex],
         xh, yh, wq, pack)
    pc["reg_ex"], pc["reg_ey"] = ex, ey
    pc["reg_core"] = _core.pair_block_contributions(*a)
    pc["reg_fallback"] = _fallback.pair_block_contributions(*a)
    # singular groups at position (2,2), T=2, N=5, p in {0, 2} on the icosphere(1)
    m1 = refine(ico, project_unit_sphere=True)
    from tdbem.assembly import classify_pair

    for p in (0, 2):
        g = TimeGrid(T=2.0, N=5, p=p)
        pk = PsiPack.build(tables_for(g), g, 2, 2)
        for case in ("coincident", "edge", "vertex"):
            pairs = []
            for e0 in range(m1.num_triangles):
                for e1 in range(m1.num_triangles):
                    c, lx, ly = classify_pair(m1, e0, e1)
                    if c == case:
                        pairs.append((e0, e1, lx, ly))
                if len(pairs) >= 24:
                    break
            pairs = pairs[:24]
            parr = np.array([(q[0], q[1]) for q in pairs])
            lx = np.array([q[2] for q in pairs])
            ly = np.array([q[3] for q in pairs])
            ax = np.arange(len(parr))
            rule = singular_rule(case, 5, 2, 2)
            args2 = (m1.corners[parr[:, 0]][ax[:, None], lx], m1.corners[parr[:, 1]][ax[:, None], ly],
                     2.0 * m1.areas[parr[:, 0]], 2.0 * m1.areas[parr[:, 1]],
                     np.einsum("pd,pd->p", m1.normals[parr[:, 0]], m1.normals[parr[:, 1]]),
                     m1.curls[parr[:, 1]][ax[:, None], ly], m1.curls[parr[:, 0]][ax[:, None], lx],
                     *rule, pk)
            pc[f"{case}_p{p}_pairs"] = parr
            pc[f"{case}_p{p}_lx"], pc[f"{case}_p{p}_ly"] = lx, ly
            pc[f"{case}_p{p}_core"] = _core.pair_block_contributions(*args2)
    np.savez_compressed(os.path.join(OUT, "pair_contrib.npz"), **pc)

    # ---- small assembled systems ----
    verts = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [1.0, 1.0, 0.5]])
    two_tri = SurfaceMesh(verts, np.array([[0, 1, 2], [1, 3, 2]]))
    cases = [
        ("two_tri_N3_p0", two_tri, TimeGrid(T=2.0, N=3, p=0)),
        ("two_tri_N4_p1", two_tri, TimeGrid(T=2.0, N=4, p=1)),
        ("two_tri_N6_p1", two_tri, TimeGrid(T=3.0, N=6, p=1)),
        ("ico_N5_p1", ico, TimeGrid(T=2.0, N=5, p=1)),
        ("sphere80_N6_p1", m1, TimeGrid(T=2.5, N=6, p=1)),
        ("ico_N8_p2", ico, TimeGrid(T=2.0, N=8, p=2)),
    ]
    for name, mesh, grid in cases:
        A = assemble_system(mesh, grid, workers=1)
        out = {"dense": reconstruct_dense(A)}
        x = np.random.default_rng(7).standard_normal(A.shape[1])
        out["x7"], out["y7"] = x, A @ x
        keys = sorted(A.unique_blocks)
        out["positions"] = np.array(keys)
        np1 = grid.p + 1
        for (kt, it) in keys:
            blocks = A.unique_blocks[(kt, it)]
            for m2 in range(np1):
                for mm1 in range(np1):
                    if blocks[m2][mm1] is not None:
                        out[f"b_{kt}_{it}_{m2}_{mm1}"] = blocks[m2][mm1].toarray()
        # direct assembly of every logical non-band position (reuse exactness oracle)
        if name in ("two_tri_N4_p1", "ico_N5_p1"):
            tabs = tables_for(grid)
            for kt in range(1, grid.N + 1):
                for it in range(1, grid.N + 1):
                    if kt - it <= -2:
                        continue
                    S = assemble_subblocks(mesh, grid, tabs, kt, it)
                    for m2 in range(np1):
                        for mm1 in range(np1):
                            out[f"direct_{kt}_{it}_{m2}_{mm1}"] = S[m2][mm1].toarray()
        np.savez_compressed(os.path.join(OUT, f"blocks_{name}.npz"), **out)
        print("wrote", name, flush=True)

    # default-config block (2,2) of two_tri at N=3 (compare with FIXTURE_BLOCK_22)
    g3 = TimeGrid(T=2.0, N=3, p=0)
    hi = assemble_subblocks(two_tri, g3, tables_for(g3), 2, 2, QuadratureConfig(8, 8, 8))[0][0].toarray()
    np.save(os.path.join(OUT, "two_tri_22_q888.npy"), hi)

    # ---- config 1 (icosphere x2, dt=0.1, N=40, p=0): selected canonical positions ----
    if not args.skip_cfg1:
        mesh = refine(refine(ico, True), True)
        grid = TimeGrid(T=3.9, N=40, p=0)
        tabs = tables_for(grid)
        mesh.tri_distance_bounds
        out = {}
        sel = [(2, 2), (2, 3), (3, 2), (9, 2), (17, 2), (24, 2), (1, 1), (1, 2), (5, 1),
               (23, 1), (39, 40), (40, 40), (40, 20), (40, 38)]
        units = []
        for kt, it in sel:
            pat = block_pattern(mesh, grid, kt, it)
            units.append(len(pat.element_pairs))
            S = assemble_subblocks(mesh, grid, tabs, kt, it)
            csr_pack(f"b_{kt}_{it}", S[0][0], out)
            print("cfg1", (kt, it), S[0][0].nnz, flush=True)
        out["positions"] = np.array(sel)
        out["units"] = np.array(units)
        # admissible-pair count of every canonical position (plan check)
        from tdbem.block_system import BlockHessenbergMatrix

        A = BlockHessenbergMatrix(grid=grid, M=mesh.num_vertices, diameter=mesh.diameter)
        allpos = set()
        for kt in range(1, grid.N + 1):
            for it in range(1, grid.N + 1):
                if A.is_zero_position(kt, it):
                    continue
                c = canonical_position(grid, kt, it)
                if c is not None:
                    allpos.add(c)
        allpos = sorted(allpos)
        out["all_positions"] = np.array(allpos)
        out["all_units"] = np.array([len(block_pattern(mesh, grid, kt, it).element_pairs) for kt, it in allpos])
        tmin, tmax = mesh.tri_distance_bounds
        sel_rows = np.array([0, 7, 100, 319])
        out["tmin_rows"], out["tmax_rows"], out["bound_rows"] = tmin[sel_rows], tmax[sel_rows], sel_rows
        np.savez_compressed(os.path.join(OUT, "blocks_cfg1.npz"), **out)


if __name__ == "__main__":
    main()
