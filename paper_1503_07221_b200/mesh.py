"""Triangle surface meshes: the SoA geometry the assembly kernel consumes.

Reference interface (``tdbem.mesh``, /root/reference/pkg/src/tdbem/mesh.py):
  SurfaceMesh.corners/areas/normals/curls   mesh.py:69-106
  SurfaceMesh.diameter                      mesh.py:108-113
  SurfaceMesh.validate_closed/signed_volume mesh.py:124-144
  load_mesh / save_mesh                     mesh.py:185-231
  icosahedron / refine                      mesh.py:234-283
The O(E^2) triangle distance bounds (mesh.py:146-168, :286-391) are NOT built
here: the device computes them pair by pair inside the assembly plan
(csrc/tdb_assembly.cu, tdb_pair_bounds), so nothing E x E lives on the host.
Also here: the seeded jittered unit-cube generator of BASELINE config 3 (not in
the reference) and the touching-pair topology the singular rules need.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from functools import cached_property

import numpy as np

__all__ = [
    "SurfaceMesh",
    "MeshError",
    "load_mesh",
    "save_mesh",
    "icosahedron",
    "refine",
    "icosphere",
    "jittered_cube",
    "touching_pairs",
]


class MeshError(ValueError):
    """Malformed mesh file or violated mesh invariant."""


@dataclass(frozen=True)
class SurfaceMesh:
    """Immutable triangle mesh; vertices (V, 3) float64, triangles (E, 3) int64."""

    vertices: np.ndarray
    triangles: np.ndarray

    def __post_init__(self):
        v = np.ascontiguousarray(np.asarray(self.vertices, dtype=np.float64))
        t = np.ascontiguousarray(np.asarray(self.triangles, dtype=np.int64))
        if v.ndim != 2 or v.shape[1] != 3:
            raise MeshError(f"vertices must have shape (M_v, 3), got {v.shape}")
        if t.ndim != 2 or t.shape[1] != 3:
            raise MeshError(f"triangles must have shape (E, 3), got {t.shape}")
        if t.size and (t.min() < 0 or t.max() >= len(v)):
            raise MeshError("triangle vertex index out of range")
        v.setflags(write=False)
        t.setflags(write=False)
        object.__setattr__(self, "vertices", v)
        object.__setattr__(self, "triangles", t)

    @property
    def num_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def num_triangles(self) -> int:
        return self.triangles.shape[0]

    @cached_property
    def corners(self) -> np.ndarray:
        """(E, 3, 3): corner a of triangle e."""
        return self.vertices[self.triangles]

    @cached_property
    def _cross(self) -> np.ndarray:
        c = self.corners
        return np.cross(c[:, 1] - c[:, 0], c[:, 2] - c[:, 0])

    @cached_property
    def areas(self) -> np.ndarray:
        return 0.5 * np.linalg.norm(self._cross, axis=1)

    @cached_property
    def normals(self) -> np.ndarray:
        n = np.linalg.norm(self._cross, axis=1)
        if np.any(n <= 0.0):
            raise MeshError("degenerate triangle (zero area)")
        return self._cross / n[:, None]

    @cached_property
    def centroids(self) -> np.ndarray:
        return self.corners.mean(axis=1)

    @cached_property
    def curls(self) -> np.ndarray:
        """(E, 3, 3): n x grad(hat_a) = (V_{a+1} - V_{a+2}) / (2 area) per flat triangle."""
        c = self.corners
        nxt = c[:, [1, 2, 0]] - c[:, [2, 0, 1]]
        return nxt / (2.0 * self.areas)[:, None, None]

    @cached_property
    def diameter(self) -> float:
        """Largest vertex-vertex distance (chunked; no V x V temporaries)."""
        v = self.vertices
        best = 0.0
        step = max(1, 4_000_000 // max(1, len(v)))
        for s in range(0, len(v), step):
            d = v[s : s + step, None, :] - v[None, :, :]
            best = max(best, float(np.sum(d * d, axis=2).max()))
        return float(np.sqrt(best))

    @cached_property
    def vertex_triangles(self) -> list[np.ndarray]:
        """Star of every vertex: ascending triangle ids containing it."""
        order = np.argsort(self.triangles.ravel(), kind="stable")
        owners = order // 3
        counts = np.bincount(self.triangles.ravel(), minlength=self.num_vertices)
        splits = np.cumsum(counts)[:-1]
        return [np.sort(s) for s in np.split(owners, splits)]

    @cached_property
    def star_csr(self) -> tuple[np.ndarray, np.ndarray]:
        """Vertex stars as CSR (offsets (V+1,), triangle ids), ascending within a star."""
        stars = self.vertex_triangles
        off = np.zeros(self.num_vertices + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(s) for s in stars])
        ids = np.concatenate(stars) if stars else np.zeros(0, dtype=np.int64)
        return off, ids.astype(np.int64)

    @cached_property
    def signed_volume(self) -> float:
        c = self.corners
        return float(np.einsum("ij,ij->", c[:, 0], np.cross(c[:, 1], c[:, 2]))) / 6.0

    def validate_closed(self) -> None:
        """Every undirected edge in exactly two triangles, once per direction."""
        t = self.triangles
        directed = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
        if len(np.unique(directed, axis=0)) != len(directed):
            raise MeshError("duplicated directed edge (inconsistent orientation)")
        _, cnt = np.unique(np.sort(directed, axis=1), axis=0, return_counts=True)
        if np.any(cnt != 2):
            raise MeshError("open or non-manifold surface (edge not shared by exactly 2 triangles)")


def load_mesh(path, validate: bool = True) -> SurfaceMesh:
    """OFF-style ASCII mesh (mesh.py:185-220 semantics, incl. the orientation flip)."""
    with open(path) as fh:
        tokens = []
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if line:
                tokens.extend(line.split())
    if not tokens or tokens[0] != "OFF":
        raise MeshError(f"{path}: missing OFF header")
    try:
        nv, ne = int(tokens[1]), int(tokens[2])
        pos = 4
        verts = np.array(tokens[pos : pos + 3 * nv], dtype=float).reshape(nv, 3)
        pos += 3 * nv
        faces = np.array(tokens[pos : pos + 4 * ne], dtype=np.int64).reshape(ne, 4)
        if faces.shape[0] != ne or len(tokens) != pos + 4 * ne:
            raise MeshError(f"{path}: trailing or missing tokens in face list")
        if np.any(faces[:, 0] != 3):
            raise MeshError(f"{path}: non-triangular face")
    except (ValueError, IndexError) as exc:
        raise MeshError(f"{path}: malformed OFF file ({exc})") from exc
    mesh = SurfaceMesh(verts, faces[:, 1:])
    mesh.normals
    if validate:
        mesh.validate_closed()
        if mesh.signed_volume < 0.0:
            warnings.warn(f"{path}: negative enclosed volume, flipping triangle orientation")
            mesh = SurfaceMesh(verts, faces[:, [1, 3, 2]])
    return mesh


def save_mesh(mesh: SurfaceMesh, path) -> None:
    with open(path, "w") as fh:
        fh.write(f"OFF\n{mesh.num_vertices} {mesh.num_triangles} 0\n")
        for x, y, z in mesh.vertices:
            fh.write(f"{x:.17g} {y:.17g} {z:.17g}\n")
        for a, b, c in mesh.triangles:
            fh.write(f"3 {a} {b} {c}\n")


def icosahedron() -> SurfaceMesh:
    """Regular icosahedron on the unit sphere, in the reference's vertex/face order."""
    g = (1.0 + np.sqrt(5.0)) / 2.0
    v = np.array([
        (-1, g, 0), (1, g, 0), (-1, -g, 0), (1, -g, 0),
        (0, -1, g), (0, 1, g), (0, -1, -g), (0, 1, -g),
        (g, 0, -1), (g, 0, 1), (-g, 0, -1), (-g, 0, 1),
    ], dtype=float)
    v /= np.linalg.norm(v[0])
    f = np.array([
        (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
        (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
        (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
        (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1),
    ], dtype=np.int64)
    return SurfaceMesh(v, f)


def refine(mesh: SurfaceMesh, project_unit_sphere: bool = False) -> SurfaceMesh:
    """1 -> 4 midpoint split; new vertices numbered in first-use order."""
    V = mesh.vertices
    new = []
    index: dict = {}
    base = len(V)

    def mid(a, b):
        key = (a, b) if a < b else (b, a)
        k = index.get(key)
        if k is None:
            k = base + len(new)
            index[key] = k
            new.append(0.5 * (V[a] + V[b]))
        return k

    out = np.empty((4 * mesh.num_triangles, 3), dtype=np.int64)
    for e, (i0, i1, i2) in enumerate(mesh.triangles.tolist()):
        a, b, c = mid(i0, i1), mid(i1, i2), mid(i2, i0)
        out[4 * e : 4 * e + 4] = ((i0, a, c), (i1, b, a), (i2, c, b), (a, b, c))
    verts = np.vstack([V, np.array(new)]) if new else V.copy()
    if project_unit_sphere:
        verts = verts / np.linalg.norm(verts, axis=1)[:, None]
    return SurfaceMesh(verts, out)


def icosphere(levels: int) -> SurfaceMesh:
    """Icosahedron refined `levels` times with projection to the unit sphere."""
    m = icosahedron()
    for _ in range(levels):
        m = refine(m, project_unit_sphere=True)
    return m


def jittered_cube(n: int = 16, jitter: float = 0.05, seed: int = 0) -> SurfaceMesh:
    """Unit cube [0,1]^3, n x n squares per face, 2 triangles each (diagonal
    (i,j)->(i+1,j+1)), outward orientation; every unique vertex jittered by a
    seeded uniform +-jitter*h in all three coordinates (BASELINE config 3).

    Vertex order: lexicographic in the integer lattice coordinates (ix, iy, iz)
    of the surface points; faces in the order -x, +x, -y, +y, -z, +z.
    """
    h = 1.0 / n
    lattice = {}
    pts = []
    for ix in range(n + 1):
        for iy in range(n + 1):
            for iz in range(n + 1):
                if ix in (0, n) or iy in (0, n) or iz in (0, n):
                    lattice[(ix, iy, iz)] = len(pts)
                    pts.append((ix * h, iy * h, iz * h))
    tris = []
    # each face: fixed axis k at level 0 or n; (u, v) the other two axes such
    # that u x v points along +k; reversed for the low face
    for k in range(3):
        u_ax, v_ax = (k + 1) % 3, (k + 2) % 3
        for level, outward in ((0, False), (n, True)):
            for i in range(n):
                for j in range(n):
                    def vid(a, b):
                        c = [0, 0, 0]
                        c[k], c[u_ax], c[v_ax] = level, a, b
                        return lattice[tuple(c)]

                    p00, p10, p11, p01 = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
                    if outward:
                        tris += [(p00, p10, p11), (p00, p11, p01)]
                    else:
                        tris += [(p00, p11, p10), (p00, p01, p11)]
    verts = np.array(pts, dtype=float)
    rng = np.random.default_rng(seed)
    verts = verts + rng.uniform(-jitter * h, jitter * h, verts.shape)
    mesh = SurfaceMesh(verts, np.array(tris, dtype=np.int64))
    mesh.validate_closed()
    if mesh.signed_volume <= 0.0:
        raise MeshError("cube generator produced inward orientation")
    return mesh


def touching_pairs(mesh: SurfaceMesh):
    """All ordered triangle pairs sharing >= 1 vertex, classified.

    Returns dict case -> (ex, ey, lx, ly) int arrays, rows sorted by (ex, ey):
    lx/ly are the chart permutations that bring the shared vertices first in
    ascending global order (assembly.py:130-152 semantics).  Vectorised over
    the vertex stars (no per-pair Python work).
    """
    tri = np.asarray(mesh.triangles, dtype=np.int64)
    off, ids = mesh.star_csr
    E = mesh.num_triangles
    # candidates: (e, f) for every f in the star of each vertex of e
    v = tri.ravel()
    cnt = off[v + 1] - off[v]
    ex = np.repeat(np.repeat(np.arange(E, dtype=np.int64), 3), cnt)
    starts = np.repeat(off[v], cnt)
    within = np.arange(len(ex), dtype=np.int64) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    ey = np.asarray(ids, dtype=np.int64)[starts + within]
    key = np.unique(ex * E + ey)
    ex, ey = key // E, key % E
    tx, ty = tri[ex], tri[ey]
    eq = tx[:, :, None] == ty[:, None, :]
    nshared = eq.sum(axis=(1, 2))
    big = np.int64(np.iinfo(np.int64).max // 4)

    def lead(t, shared):
        # shared vertices first in ascending global id, then the rest in local order
        k = np.where(shared, t, big + np.arange(3, dtype=np.int64)[None, :])
        return np.argsort(k, axis=1, kind="stable").astype(np.int64)

    lx = lead(tx, eq.any(axis=2))
    ly = lead(ty, eq.any(axis=1))
    coinc = ex == ey
    lx[coinc] = (0, 1, 2)
    ly[coinc] = (0, 1, 2)
    res = {}
    for case, sel in (("coincident", coinc), ("edge", ~coinc & (nshared == 2)), ("vertex", ~coinc & (nshared == 1))):
        res[case] = (ex[sel], ey[sel], lx[sel].reshape(-1, 3), ly[sel].reshape(-1, 3))
    return res


def _touching_pairs_loop(mesh: SurfaceMesh):
    """Per-pair reference restatement of touching_pairs (kept for tests)."""
    tri = mesh.triangles
    off, ids = mesh.star_csr
    E = mesh.num_triangles
    cand = set()
    for e in range(E):
        for v in tri[e]:
            for f in ids[off[v] : off[v + 1]]:
                cand.add((e, int(f)))
    pairs = sorted(cand)
    out = {c: ([], [], [], []) for c in ("coincident", "edge", "vertex")}
    for ex, ey in pairs:
        tx, ty = tri[ex].tolist(), tri[ey].tolist()
        if ex == ey:
            case, lx, ly = "coincident", (0, 1, 2), (0, 1, 2)
        else:
            shared = sorted(set(tx) & set(ty))
            lx = _lead(tx, shared)
            ly = _lead(ty, shared)
            case = "edge" if len(shared) == 2 else "vertex"
        o = out[case]
        o[0].append(ex)
        o[1].append(ey)
        o[2].append(lx)
        o[3].append(ly)
    res = {}
    for c, (ex, ey, lx, ly) in out.items():
        res[c] = (
            np.array(ex, dtype=np.int64),
            np.array(ey, dtype=np.int64),
            np.array(lx, dtype=np.int64).reshape(-1, 3),
            np.array(ly, dtype=np.int64).reshape(-1, 3),
        )
    return res


def _lead(t, shared):
    lead = [t.index(g) for g in shared]
    return tuple(lead + [a for a in range(3) if a not in lead])
