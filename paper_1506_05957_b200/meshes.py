"""Closed triangulated surfaces for the five benchmark configurations.

This is input generation, not the hot path.  The reference only refines an
octahedron (``pkg/src/fmmbem/mesh.py:75-118``); BASELINE.json asks for
icospheres (20 * 4**L panels) and for a 64-cell red-blood-cell lattice, so
both generators are new here.  The biconcave-disc map follows the published
Evans-Fung profile the reference uses (``mesh.py:121-145``) and the ASCII
interchange format matches ``mesh.py:175-200`` so meshes can round-trip
between this package and the reference oracle.

Every generator is deterministic: the same arguments give bit-identical
vertex and triangle arrays, which is what makes the octree (and therefore the
mat-vec) reproducible across the GPU path and the CPU oracle.
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field

import numpy as np

GOLDEN = (1.0 + 5.0 ** 0.5) / 2.0


@dataclass
class Mesh:
    """Vertices (V, 3) float64 and outward-oriented triangles (P, 3) int64."""

    vertices: np.ndarray
    triangles: np.ndarray
    tags: np.ndarray = field(default=None)

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64)
        self.triangles = np.ascontiguousarray(self.triangles, dtype=np.int64)
        if self.vertices.ndim != 2 or self.vertices.shape[1] != 3:
            raise ValueError("vertices must be (V, 3)")
        if self.triangles.ndim != 2 or self.triangles.shape[1] != 3:
            raise ValueError("triangles must be (P, 3)")
        if len(self.triangles) and (self.triangles.min() < 0
                                    or self.triangles.max() >= len(self.vertices)):
            raise ValueError("triangle indices out of range")
        if self.tags is None:
            self.tags = np.zeros(len(self.triangles), dtype=np.int64)
        else:
            self.tags = np.asarray(self.tags, dtype=np.int64)
            if self.tags.shape != (len(self.triangles),):
                raise ValueError("tags must have one entry per triangle")

    @property
    def n_panels(self) -> int:
        return int(len(self.triangles))

    @property
    def panel_vertices(self) -> np.ndarray:
        return self.vertices[self.triangles]

    def geometry(self):
        from .geometry import panel_geometry
        return panel_geometry(self.panel_vertices)

    @property
    def volume(self) -> float:
        v = self.panel_vertices
        return float(np.einsum("pi,pi->p", v[:, 0], np.cross(v[:, 1], v[:, 2])).sum() / 6.0)


def _refine(vertices: np.ndarray, triangles: np.ndarray):
    """One 1-to-4 split through deduplicated edge midpoints (vectorised).

    New vertices are appended in order of first appearance of their edge in
    the (triangle, edge) scan, so the output is a pure function of the input.
    """
    a, b, c = triangles[:, 0], triangles[:, 1], triangles[:, 2]
    edges = np.stack([np.stack([a, b], 1), np.stack([b, c], 1), np.stack([c, a], 1)], 1)
    flat = np.sort(edges.reshape(-1, 2), axis=1)
    nv = len(vertices)
    key = flat[:, 0] * nv + flat[:, 1]
    uniq, first, inverse = np.unique(key, return_index=True, return_inverse=True)
    # number midpoints by first appearance, not by key order
    order = np.argsort(first, kind="stable")
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    mid_id = nv + rank[inverse.ravel()]
    lo = uniq[order] // nv
    hi = uniq[order] % nv
    mids = 0.5 * (vertices[lo] + vertices[hi])
    m = mid_id.reshape(-1, 3)
    ab, bc, ca = m[:, 0], m[:, 1], m[:, 2]
    tris = np.stack([
        np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
        np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], 1).reshape(-1, 3)
    return np.vstack([vertices, mids]), tris


def _outward(vertices: np.ndarray, faces: np.ndarray) -> np.ndarray:
    """Orient faces of a convex, origin-centred polyhedron outward."""
    v = vertices[faces]
    n = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
    flip = np.einsum("fi,fi->f", n, v.mean(axis=1)) < 0.0
    faces = faces.copy()
    faces[flip] = faces[flip][:, [0, 2, 1]]
    return faces


def _icosahedron():
    pts = []
    for s1 in (-1.0, 1.0):
        for s2 in (-1.0, 1.0):
            pts.append((0.0, s1, s2 * GOLDEN))
            pts.append((s1, s2 * GOLDEN, 0.0))
            pts.append((s2 * GOLDEN, 0.0, s1))
    verts = np.asarray(pts)
    # faces = triples of mutually adjacent vertices (edge length 2)
    d = np.linalg.norm(verts[:, None] - verts[None], axis=-1)
    adj = np.abs(d - 2.0) < 1e-9
    faces = [(i, j, k) for i in range(12) for j in range(i + 1, 12) for k in range(j + 1, 12)
             if adj[i, j] and adj[j, k] and adj[i, k]]
    faces = _outward(verts, np.asarray(faces, dtype=np.int64))
    return verts / np.linalg.norm(verts, axis=1, keepdims=True), faces


def _octahedron():
    verts = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]],
                     dtype=np.float64)
    faces = [(i, j, k) for i in (0, 1) for j in (2, 3) for k in (4, 5)]
    return verts, _outward(verts, np.asarray(faces, dtype=np.int64))


def _refined_sphere(base, level: int):
    if level < 0:
        raise ValueError("level must be >= 0")
    verts, tris = base
    for _ in range(level):
        verts, tris = _refine(verts, tris)
        verts = verts / np.linalg.norm(verts, axis=1, keepdims=True)
    return verts, tris


def make_icosphere(level: int, radius: float = 1.0, center=(0.0, 0.0, 0.0)) -> Mesh:
    """Unit-sphere icosphere with 20 * 4**level panels (BASELINE configs 1, 2, 3, 5)."""
    verts, tris = _refined_sphere(_icosahedron(), level)
    return Mesh(verts * radius + np.asarray(center, dtype=np.float64), tris)


def make_octasphere(level: int, radius: float = 1.0, center=(0.0, 0.0, 0.0)) -> Mesh:
    """Octahedral sphere with 8 * 4**level panels (the reference's sphere family)."""
    verts, tris = _refined_sphere(_octahedron(), level)
    return Mesh(verts * radius + np.asarray(center, dtype=np.float64), tris)


RBC_SCALE = 3.91
RBC_SHAPE = (0.81, 7.83, -4.39)


def rbc_transform(points, scale=RBC_SCALE, shape=RBC_SHAPE):
    """Evans-Fung biconcave profile: z = +-1/2 sqrt(1-s^2)(C0 + C2 s^2 + C4 s^4), s = rho/scale."""
    p = np.asarray(points, dtype=np.float64) * scale
    c0, c2, c4 = shape
    s2 = np.clip((p[:, 0] ** 2 + p[:, 1] ** 2) / scale ** 2, 0.0, 1.0)
    z = 0.5 * np.sqrt(1.0 - s2) * (c0 + c2 * s2 + c4 * s2 ** 2)
    out = p.copy()
    out[:, 2] = np.sign(p[:, 2]) * z
    return out


def make_rbc(level: int = 4) -> Mesh:
    """One biconcave cell (2048 panels at level 4)."""
    s = make_octasphere(level)
    return Mesh(rbc_transform(s.vertices), s.triangles)


def make_rbc_lattice(n_side: int = 4, level: int = 4, gap: float = 1.0, seed: int = 0) -> Mesh:
    """n_side**3 randomly rotated cells on a cubic lattice (BASELINE config 4).

    Pitch = cell diameter + gap, i.e. ``gap`` microns between bounding spheres.
    """
    from scipy.spatial.transform import Rotation

    rng = np.random.default_rng(seed)
    cell = make_rbc(level)
    pitch = 2.0 * RBC_SCALE + gap
    verts, tris = [], []
    off = 0
    for i in range(n_side):
        for j in range(n_side):
            for k in range(n_side):
                rot = Rotation.random(rng=rng)
                v = rot.apply(cell.vertices) + pitch * np.array([i, j, k], dtype=np.float64)
                verts.append(v)
                tris.append(cell.triangles + off)
                off += len(v)
    return Mesh(np.vstack(verts), np.vstack(tris))


def write_mesh(path, mesh: Mesh) -> None:
    """ASCII: 'nv np' header, nv vertex lines (%.17g), np 'i j k tag' lines."""
    buf = io.StringIO()
    buf.write(f"{len(mesh.vertices)} {mesh.n_panels}\n")
    np.savetxt(buf, mesh.vertices, fmt="%.17g")
    np.savetxt(buf, np.column_stack([mesh.triangles, mesh.tags]), fmt="%d")
    with open(path, "w") as fh:
        fh.write(buf.getvalue())


def read_mesh(path) -> Mesh:
    with open(path) as fh:
        nv, npan = map(int, fh.readline().split())
        verts = np.loadtxt(fh, max_rows=nv, ndmin=2)
        tris = np.loadtxt(fh, dtype=np.int64, max_rows=npan, ndmin=2)
    if verts.shape != (nv, 3) or tris.shape[0] != npan or tris.shape[1] not in (3, 4):
        raise ValueError("mesh file does not match its header counts")
    tags = tris[:, 3] if tris.shape[1] == 4 else None
    return Mesh(verts, tris[:, :3], tags)


def is_closed(mesh: Mesh) -> bool:
    """Every directed edge appears once and its reverse appears once."""
    t = mesh.triangles
    e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    nv = len(mesh.vertices)
    fwd = e[:, 0] * nv + e[:, 1]
    rev = e[:, 1] * nv + e[:, 0]
    if len(np.unique(fwd)) != len(fwd):
        return False
    return bool(np.all(np.isin(rev, fwd)))
