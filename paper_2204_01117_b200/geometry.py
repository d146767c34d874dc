"""Closed triangle meshes for the voxelizer (reference ``citywind.geometry``).

Mesh *construction* stays on the host (it is O(#triangles) setup, like the
reference's): ``TriangleMesh``, ``box_mesh``, ``cylinder_mesh``, ``load_obj``,
``mesh_aabb``.  The inside/outside classification of sample points -- the
O(cells x samples x triangles) part -- runs on the device inside
``cw_voxelize`` (csrc/cw_voxel.cu).  Vertex coordinates are produced with
the same numpy expressions as the reference (geometry.py:276-316), so the
device sees bit-identical triangles.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

from .errors import ClassificationError, MeshError

_CLOSED = set()   # triangle connectivities already shown to be closed

__all__ = ["TriangleMesh", "Aabb", "mesh_aabb", "box_mesh", "cylinder_mesh", "load_obj",
           "MeshError", "ClassificationError"]


@dataclass(frozen=True)
class Aabb:
    min: np.ndarray
    max: np.ndarray

    def contains(self, points):
        p = np.atleast_2d(points)
        return np.all((p >= self.min) & (p <= self.max), axis=1)

    def expanded(self, margin):
        return Aabb(self.min - margin, self.max + margin)


class TriangleMesh:
    """Indexed triangle surface (geometry.py:70-105)."""

    def __init__(self, vertices, triangles):
        self.vertices = np.asarray(vertices, dtype=float).reshape(-1, 3)
        self.triangles = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
        if len(self.vertices) == 0 or len(self.triangles) == 0:
            raise MeshError("empty mesh")
        if self.triangles.min() < 0 or self.triangles.max() >= len(self.vertices):
            raise MeshError("triangle vertex index out of range")

    def validate_closed(self):
        t = self.triangles
        key = hashlib.sha1(np.ascontiguousarray(t).tobytes()).digest()
        if key in _CLOSED:         # closedness depends on the connectivity only
            return
        edges = np.sort(np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]]), axis=1)
        _, counts = np.unique(edges, axis=0, return_counts=True)
        if np.any(counts != 2):
            raise MeshError(f"mesh is not closed: {int(np.sum(counts != 2))} edges not shared "
                            "by exactly 2 triangles")
        _CLOSED.add(key)

    def translated(self, offset):
        return TriangleMesh(self.vertices + np.asarray(offset, dtype=float), self.triangles.copy())


def mesh_aabb(mesh: TriangleMesh) -> Aabb:
    return Aabb(mesh.vertices.min(axis=0), mesh.vertices.max(axis=0))


def box_mesh(lo, hi) -> TriangleMesh:
    """Closed axis-aligned box (outward faces)."""
    x0, y0, z0 = np.asarray(lo, dtype=float)
    x1, y1, z1 = np.asarray(hi, dtype=float)
    v = np.array([[x0, y0, z0], [x1, y0, z0], [x1, y1, z0], [x0, y1, z0],
                  [x0, y0, z1], [x1, y0, z1], [x1, y1, z1], [x0, y1, z1]])
    quads = np.array([(0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4),
                      (2, 3, 7, 6), (0, 4, 7, 3), (1, 2, 6, 5)])
    tris = np.concatenate([quads[:, [0, 1, 2]], quads[:, [0, 2, 3]]], axis=1).reshape(-1, 3)
    return TriangleMesh(v, tris)


def cylinder_mesh(center, radius, z0, z1, segments: int = 48) -> TriangleMesh:
    """Closed vertical cylinder with fan caps: ring vertices at the bottom and
    the top, then the two cap centres; four triangles per segment."""
    cx, cy = center
    ang = np.linspace(0.0, 2 * np.pi, segments, endpoint=False)
    xr = cx + radius * np.cos(ang)
    yr = cy + radius * np.sin(ang)
    verts = np.empty((2 * segments + 2, 3))
    verts[:segments, 0], verts[:segments, 1], verts[:segments, 2] = xr, yr, z0
    verts[segments:2 * segments, 0] = xr
    verts[segments:2 * segments, 1] = yr
    verts[segments:2 * segments, 2] = z1
    verts[-2] = (cx, cy, z0)
    verts[-1] = (cx, cy, z1)
    i = np.arange(segments)
    j = (i + 1) % segments
    bot, top = 2 * segments, 2 * segments + 1
    quad = np.stack([
        np.stack([i, j, segments + j], 1),
        np.stack([i, segments + j, segments + i], 1),
        np.stack([np.full(segments, bot), j, i], 1),
        np.stack([np.full(segments, top), segments + i, segments + j], 1)], 1)
    return TriangleMesh(verts, quad.reshape(-1, 3))


def load_obj(path) -> TriangleMesh:
    """'v' and 'f' records of a Wavefront OBJ; polygons are fanned."""
    vertices, faces = [], []
    with open(path) as fh:
        for line in fh:
            parts = line.split()
            if not parts or parts[0].startswith("#"):
                continue
            if parts[0] == "v":
                vertices.append([float(x) for x in parts[1:4]])
            elif parts[0] == "f":
                ids = [int(tok.split("/")[0]) for tok in parts[1:]]
                ids = [i - 1 if i > 0 else len(vertices) + i for i in ids]
                faces.extend([ids[0], a, b] for a, b in zip(ids[1:-1], ids[2:]))
    if not vertices or not faces:
        raise MeshError(f"{path}: no usable v/f records")
    mesh = TriangleMesh(np.array(vertices), np.array(faces))
    mesh.validate_closed()
    return mesh
