"""Host-side surface meshes: the input data of the per-frequency solve.

Mesh construction is setup, not hot path ("Mesh": out of
scope as a kernel).  It still has to live here because the reference
package does not exist on the GPU box, and the derived geometry must be
bit-identical to the reference's so that the tier classification of
element pairs (a last-bit decision on box meshes)
reproduces.  Every expression below uses the same numpy operations in the
same order as the reference:

* derived geometry   — reference ``mesh.py:88-106``
* box generator      — reference ``mesh.py:279-344``
* icosphere          — reference ``mesh.py:347-404`` (vertices normalised
  once at the end, never per level: App. B-7)
* merge              — reference ``mesh.py:407-424``

The generators are verified bit-for-bit against the live reference in
``tests/test_mesh_host.py`` and against committed hashes in
``tests/golden``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BOX_FACE_NAMES = ("x-", "x+", "y-", "y+", "z-", "z+")
DEGENERATE_AREA_REL = 1e-14


class MeshError(ValueError):
    """Invalid mesh topology or geometry (reference ``mesh.py:28``)."""


@dataclass
class TriangleMesh:
    """Closed flat-triangle surface with derived per-element geometry.

    Same fields and meaning as the reference ``TriangleMesh``
    (``mesh.py:37-80``): ``centroids``, unit ``normals`` (outward for a
    solid, inward for ``flip=True`` cavities), ``areas`` and
    ``diameters`` (longest edge).
    """

    vertices: np.ndarray
    triangles: np.ndarray
    region_tag: np.ndarray | None = None
    closed: bool = True
    centroids: np.ndarray = field(init=False, repr=False)
    normals: np.ndarray = field(init=False, repr=False)
    areas: np.ndarray = field(init=False, repr=False)
    diameters: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64)
        self.triangles = np.ascontiguousarray(self.triangles, dtype=np.int64)
        if self.region_tag is None:
            self.region_tag = np.zeros(len(self.triangles), dtype=np.int64)
        self.region_tag = np.ascontiguousarray(self.region_tag, dtype=np.int64)
        if len(self.triangles) == 0:
            raise MeshError("mesh has no triangles")
        if self.triangles.min() < 0 or self.triangles.max() >= len(self.vertices):
            raise MeshError("triangle vertex index out of range")
        self._derive()
        self._check()

    @property
    def n_elements(self) -> int:
        return len(self.triangles)

    @property
    def n_dofs(self) -> int:
        return 3 * len(self.triangles)

    def element_vertices(self, e: int) -> np.ndarray:
        return self.vertices[self.triangles[e]]

    def corner_arrays(self):
        """(v0, v1, v2), each (n_e, 3) float64."""
        t = self.triangles
        return self.vertices[t[:, 0]], self.vertices[t[:, 1]], self.vertices[t[:, 2]]

    def _derive(self) -> None:
        p0, p1, p2 = self.corner_arrays()
        e01 = p1 - p0
        e02 = p2 - p0
        cr = np.cross(e01, e02)
        twice_area = np.linalg.norm(cr, axis=1)
        self.areas = 0.5 * twice_area
        with np.errstate(invalid="ignore", divide="ignore"):
            self.normals = cr / twice_area[:, None]
        self.centroids = (p0 + p1 + p2) / 3.0
        lengths = np.stack([np.linalg.norm(p1 - p0, axis=1),
                            np.linalg.norm(p2 - p1, axis=1),
                            np.linalg.norm(p0 - p2, axis=1)], axis=1)
        self.diameters = lengths.max(axis=1)

    def _check(self) -> None:
        t = self.triangles
        if ((t[:, 0] == t[:, 1]) | (t[:, 1] == t[:, 2]) | (t[:, 2] == t[:, 0])).any():
            raise MeshError("triangle repeats a vertex index")
        if not np.isfinite(self.vertices).all():
            raise MeshError("non-finite vertex coordinates")
        mean_area = float(self.areas.mean())
        if (self.areas <= DEGENERATE_AREA_REL * mean_area).any():
            raise MeshError("degenerate triangle")
        if self.closed:
            directed = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
            keys = directed[:, 0] * (len(self.vertices) + 1) + directed[:, 1]
            if len(np.unique(keys)) != len(keys):
                raise MeshError("directed edge occurs twice (fold or overlap)")
            rev = directed[:, 1] * (len(self.vertices) + 1) + directed[:, 0]
            if not np.isin(rev, keys).all():
                raise MeshError("mesh is not a closed manifold")


def generate_box_mesh(lengths, divisions) -> TriangleMesh:
    """Box [0,Lx]x[0,Ly]x[0,Lz], faces tagged x-,x+,y-,y+,z-,z+ = 0..5.

    Vertex numbering, face order and the quad split follow the reference
    generator exactly (``mesh.py:279-344``) so element indices match.
    """
    lengths = [float(v) for v in lengths]
    divisions = [int(v) for v in divisions]
    if min(lengths) <= 0:
        raise ValueError("box lengths must be positive")
    if min(divisions) < 1:
        raise ValueError("box divisions must be >= 1")
    step = [lengths[a] / divisions[a] for a in range(3)]
    index: dict = {}
    coords: list = []

    def vertex(ijk):
        got = index.get(ijk)
        if got is None:
            got = index[ijk] = len(coords)
            coords.append((ijk[0] * step[0], ijk[1] * step[1], ijk[2] * step[2]))
        return got

    # (normal axis, lattice plane, in-plane axis a, in-plane axis b):
    # unit(a) x unit(b) is the outward normal of the face.
    face_specs = ((0, 0, 2, 1), (0, divisions[0], 1, 2),
                  (1, 0, 0, 2), (1, divisions[1], 2, 0),
                  (2, 0, 1, 0), (2, divisions[2], 0, 1))
    tris, tags = [], []
    for tag, (fixed, plane, ax_a, ax_b) in enumerate(face_specs):
        for a in range(divisions[ax_a]):
            for b in range(divisions[ax_b]):
                corner = []
                for da, db in ((0, 0), (1, 0), (1, 1), (0, 1)):
                    ijk = [0, 0, 0]
                    ijk[fixed] = plane
                    ijk[ax_a] = a + da
                    ijk[ax_b] = b + db
                    corner.append(vertex(tuple(ijk)))
                tris.append((corner[0], corner[1], corner[2]))
                tris.append((corner[0], corner[2], corner[3]))
                tags += [tag, tag]
    return TriangleMesh(np.array(coords, dtype=np.float64),
                        np.array(tris, dtype=np.int64),
                        np.array(tags, dtype=np.int64), closed=True)


_ICO_TRIS = (
    (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
    (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
    (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
    (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1),
)


def _split_all(verts: list, tris):
    """One midpoint subdivision level; new midpoints appended in first-use order."""
    cache: dict = {}

    def midpoint(a, b):
        key = (a, b) if a < b else (b, a)
        got = cache.get(key)
        if got is None:
            got = cache[key] = len(verts)
            verts.append(tuple((np.array(verts[a]) + np.array(verts[b])) / 2.0))
        return got

    out = []
    for a, b, c in tris:
        ab, bc, ca = midpoint(a, b), midpoint(b, c), midpoint(c, a)
        out += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
    return out


def generate_icosphere(center, radius: float, subdivisions: int = 1,
                       flip: bool = False, region_tag: int = 0) -> TriangleMesh:
    """Icosphere; ``flip=True`` reverses winding (normals toward the centre)."""
    g = (1.0 + np.sqrt(5.0)) / 2.0
    base = np.array([(-1, g, 0), (1, g, 0), (-1, -g, 0), (1, -g, 0),
                     (0, -1, g), (0, 1, g), (0, -1, -g), (0, 1, -g),
                     (g, 0, -1), (g, 0, 1), (-g, 0, -1), (-g, 0, 1)],
                    dtype=np.float64)
    verts = list(map(tuple, base))
    tris = list(_ICO_TRIS)
    for _ in range(max(0, int(subdivisions))):
        tris = _split_all(verts, tris)
    v = np.array(verts, dtype=np.float64)
    v = v / np.linalg.norm(v, axis=1)[:, None]
    v = np.asarray(center, dtype=float) + radius * v
    t = np.array(tris, dtype=np.int64)
    if flip:
        t = t[:, [0, 2, 1]]
    return TriangleMesh(v, t, np.full(len(t), region_tag, dtype=np.int64), closed=True)


def merge_meshes(meshes) -> TriangleMesh:
    meshes = list(meshes)
    if not meshes:
        raise ValueError("no meshes to merge")
    verts, tris, tags, base = [], [], [], 0
    for m in meshes:
        verts.append(m.vertices)
        tris.append(m.triangles + base)
        tags.append(m.region_tag)
        base += len(m.vertices)
    return TriangleMesh(np.concatenate(verts), np.concatenate(tris),
                        np.concatenate(tags), closed=all(m.closed for m in meshes))
