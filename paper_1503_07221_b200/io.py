"""On-disk and in-memory formats either side of the assembly / solve path
(SURVEY 8(f) row 4).

  to_reference_matrix    the assembled blocks as the reference's own
                         tdbem.block_system.BlockHessenbergMatrix (block_system.py:130-146:
                         grid, M, diameter, unique_blocks, plan), so reference code
                         (its matvec, solvers, reconstruct_dense) runs on them
  matrix_statistics /    the optional matrix-statistics dump of SPEC.md:411: one row
  write_matrix_statistics_csv   per structurally non-zero logical block position
                         (kt, it), its canonical key, stored nnz and owner rank
  save_coefficients      coefficients.npy as the reference CLI writes it (cli.py:356)
  write_vtu              ASCII VTK XML unstructured grid with one point array
                         'u_total' (the reference's field writer format, cli.py:268-309)
"""

from __future__ import annotations

import csv

import numpy as np

from .block_system import canonical_position

__all__ = ["to_reference_matrix", "matrix_statistics", "write_matrix_statistics_csv", "save_coefficients",
           "write_vtu"]


def to_reference_matrix(A, tdbem=None):
    """A (BlockHessenbergMatrix of this package) as a tdbem BlockHessenbergMatrix.

    `tdbem` is the reference package (imported when None).  The stored blocks are
    the same scipy CSR objects as A.unique_blocks (reference layout: inner
    positions keep m1 <= m2)."""
    if tdbem is None:
        import tdbem  # noqa: F401
        import tdbem.block_system
        import tdbem.temporal_basis
    bs, tb = tdbem.block_system, tdbem.temporal_basis
    grid = tb.TimeGrid(T=A.grid.T, N=A.grid.N, p=A.grid.p)
    return bs.BlockHessenbergMatrix(grid=grid, M=A.M, diameter=A.diameter, unique_blocks=dict(A.unique_blocks),
                                    plan=None)


def matrix_statistics(A, plan=None) -> list:
    """Rows (kt, it, canonical_kt, canonical_it, nnz, owner) for every structurally
    non-zero logical block position, in (kt, it) order.  nnz counts the stored
    entries of the canonical block (all (p+1)^2 sub-blocks, explicit zeros included);
    owner is the rank of the canonical position in `plan` (-1 without a plan)."""
    g = A.grid
    stored = A.unique_blocks
    nnz = {pos: sum(b.nnz for row in blocks for b in row if b is not None) for pos, blocks in stored.items()}
    rows = []
    for kt in range(1, g.N + 1):
        for it in range(1, g.N + 1):
            if A.is_zero_position(kt, it):
                continue
            pos = canonical_position(g, kt, it)
            if pos is None or pos not in stored:
                continue
            owner = -1
            if plan is not None:
                owner = int(plan.owners.get(pos, -1))
            rows.append((kt, it, pos[0], pos[1], int(nnz[pos]), owner))
    return rows


def write_matrix_statistics_csv(A, path: str, plan=None) -> int:
    """Write matrix_statistics as CSV (header row, comma separated)."""
    rows = matrix_statistics(A, plan)
    with open(path, "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(["kt", "it", "canonical_kt", "canonical_it", "nnz", "owner"])
        wr.writerows(rows)
    return len(rows)


def save_coefficients(path: str, x) -> None:
    """Solution vector (time-major, L * M) as coefficients.npy (cli.py:356)."""
    arr = x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)
    np.save(path, np.asarray(arr, dtype=np.float64))


def write_vtu(path: str, points, values, dims=None) -> None:
    """ASCII VTU with point array 'u_total'; dims = (n1, n2) -> quad cells of a
    structured slice (row-major point order), else vertex cells."""
    points = np.atleast_2d(np.asarray(points, dtype=float))
    npts = len(points)
    if dims is not None:
        n1, n2 = dims
        a, b = np.meshgrid(np.arange(n1 - 1), np.arange(n2 - 1), indexing="ij")
        base = (a * n2 + b).ravel()
        cells = np.stack([base, base + n2, base + n2 + 1, base + 1], axis=1)
        ctype = 9  # VTK_QUAD
    else:
        cells = np.arange(npts)[:, None]
        ctype = 1  # VTK_VERTEX
    offs = np.cumsum(np.full(len(cells), cells.shape[1]))
    with open(path, "w") as fh:
        fh.write('<?xml version="1.0"?>\n')
        fh.write('<VTKFile type="UnstructuredGrid" version="0.1" byte_order="LittleEndian">\n')
        fh.write(f'<UnstructuredGrid><Piece NumberOfPoints="{npts}" NumberOfCells="{len(cells)}">\n')
        fh.write('<Points><DataArray type="Float64" NumberOfComponents="3" format="ascii">\n')
        fh.writelines(f"{p[0]:.12g} {p[1]:.12g} {p[2]:.12g}\n" for p in points)
        fh.write('</DataArray></Points>\n<Cells>\n')
        fh.write('<DataArray type="Int64" Name="connectivity" format="ascii">\n')
        fh.writelines(" ".join(str(int(i)) for i in c) + "\n" for c in cells)
        fh.write('</DataArray>\n<DataArray type="Int64" Name="offsets" format="ascii">\n')
        fh.write(" ".join(str(int(o)) for o in offs) + "\n")
        fh.write('</DataArray>\n<DataArray type="UInt8" Name="types" format="ascii">\n')
        fh.write(" ".join(str(ctype) for _ in range(len(cells))) + "\n")
        fh.write('</DataArray>\n</Cells>\n')
        fh.write('<PointData Scalars="u_total">\n')
        fh.write('<DataArray type="Float64" Name="u_total" format="ascii">\n')
        fh.writelines(f"{v:.12g}\n" for v in np.asarray(values, dtype=float).ravel())
        fh.write('</DataArray>\n</PointData>\n</Piece></UnstructuredGrid></VTKFile>\n')
