"""Surface-mesh input of the device path.

Meshes are inputs, not part of the hot path (generation and I/O
are out of scope).  ``Assembler`` accepts any object with the reference
``TriangleMesh`` fields (``vertices``, ``triangles``, ``region_tag``,
``centroids``, ``normals``, ``areas``, ``diameters``, ``n_elements``,
``n_dofs``; reference ``mesh.py:37-106``) — in particular the reference's
own meshes.  ``SurfaceMesh`` is the minimal stand-in used where the
reference does not exist (the GPU box): it takes vertex / triangle arrays
(the tests and the benchmark load reference-generated ones from
``tests/golden/meshes.npz``) and derives the per-element geometry with the
same numpy operations as ``mesh.py:88-106``, so the last-bit tier decisions
of the box meshes reproduce; ``tests/test_host.py``
checks the derivation bitwise against the reference's values.
"""

from __future__ import annotations

import numpy as np


class SurfaceMesh:
    """Flat-triangle surface with derived per-element geometry."""

    def __init__(self, vertices, triangles, region_tag=None):
        self.vertices = np.ascontiguousarray(vertices, dtype=np.float64)
        self.triangles = np.ascontiguousarray(triangles, dtype=np.int64)
        if self.triangles.ndim != 2 or self.triangles.shape[1] != 3 or not len(self.triangles):
            raise ValueError("triangles must be a non-empty (n, 3) index array")
        if self.triangles.min() < 0 or self.triangles.max() >= len(self.vertices):
            raise ValueError("triangle vertex index out of range")
        self.region_tag = (np.zeros(len(self.triangles), dtype=np.int64) if region_tag is None
                           else np.ascontiguousarray(region_tag, dtype=np.int64))
        corner = [self.vertices[self.triangles[:, c]] for c in range(3)]
        cross = np.cross(corner[1] - corner[0], corner[2] - corner[0])
        double_area = np.linalg.norm(cross, axis=1)
        self.areas = 0.5 * double_area
        with np.errstate(invalid="ignore", divide="ignore"):
            self.normals = cross / double_area[:, None]
        self.centroids = (corner[0] + corner[1] + corner[2]) / 3.0
        edges = np.stack([np.linalg.norm(corner[1] - corner[0], axis=1),
                          np.linalg.norm(corner[2] - corner[1], axis=1),
                          np.linalg.norm(corner[0] - corner[2], axis=1)], axis=1)
        self.diameters = edges.max(axis=1)

    @property
    def n_elements(self) -> int:
        return len(self.triangles)

    @property
    def n_dofs(self) -> int:
        return 3 * len(self.triangles)


def corner_arrays(mesh):
    """(v0, v1, v2), each (n_e, 3) float64, of any TriangleMesh-like object."""
    v = np.asarray(mesh.vertices, dtype=np.float64)
    t = np.asarray(mesh.triangles)
    return v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
