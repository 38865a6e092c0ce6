"""Host-side mesh container mirroring ``meshforge::TriangleMesh``.

Reference: ``proj/include/meshforge/core/mesh.h:15-26``. Positions and normals
are float64 ``(V, 3)``, faces int32 ``(F, 3)``, UVs float64 ``(U, 2)`` in a
separate pool indexed per corner by ``face_uvs`` int32 ``(F, 3)``. The arrays
are C-contiguous so they pass to the C ABI (``include/mfbake.h``) as the same
bytes ``std::vector<Eigen::Vector3d>::data()`` would.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np


class MfMeshView(ctypes.Structure):
    """``mf_mesh_view`` from include/mfbake.h."""

    _fields_ = [
        ("positions", ctypes.POINTER(ctypes.c_double)),
        ("n_vertices", ctypes.c_int32),
        ("faces", ctypes.POINTER(ctypes.c_int32)),
        ("n_faces", ctypes.c_int32),
        ("normals", ctypes.POINTER(ctypes.c_double)),
        ("uvs", ctypes.POINTER(ctypes.c_double)),
        ("n_uvs", ctypes.c_int32),
        ("face_uvs", ctypes.POINTER(ctypes.c_int32)),
    ]


def _dptr(a: Optional[np.ndarray]):
    if a is None or a.size == 0:
        return ctypes.POINTER(ctypes.c_double)()
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _iptr(a: Optional[np.ndarray]):
    if a is None or a.size == 0:
        return ctypes.POINTER(ctypes.c_int32)()
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


@dataclass
class TriangleMesh:
    positions: np.ndarray
    faces: np.ndarray
    normals: Optional[np.ndarray] = None
    uvs: Optional[np.ndarray] = None
    face_uvs: Optional[np.ndarray] = None
    _keep: list = field(default_factory=list, repr=False, compare=False)

    def __post_init__(self):
        self.positions = np.ascontiguousarray(np.asarray(self.positions, dtype=np.float64).reshape(-1, 3))
        self.faces = np.ascontiguousarray(np.asarray(self.faces, dtype=np.int32).reshape(-1, 3))
        if self.normals is not None:
            self.normals = np.ascontiguousarray(np.asarray(self.normals, dtype=np.float64).reshape(-1, 3))
        if self.uvs is not None:
            self.uvs = np.ascontiguousarray(np.asarray(self.uvs, dtype=np.float64).reshape(-1, 2))
        if self.face_uvs is not None:
            self.face_uvs = np.ascontiguousarray(np.asarray(self.face_uvs, dtype=np.int32).reshape(-1, 3))

    # mesh.h:21-25
    def vertex_count(self) -> int:
        return int(self.positions.shape[0])

    def face_count(self) -> int:
        return int(self.faces.shape[0])

    def has_normals(self) -> bool:
        return self.normals is not None and self.normals.shape[0] == self.positions.shape[0] > 0

    def has_uvs(self) -> bool:
        return (self.face_uvs is not None and self.uvs is not None
                and self.face_uvs.shape[0] == self.faces.shape[0] and self.uvs.shape[0] > 0)

    def bounds(self):
        """``bounds(mesh)`` (mesh.cpp:12-16) as (min, max)."""
        return self.positions.min(axis=0), self.positions.max(axis=0)

    def bbox_diagonal(self) -> float:
        lo, hi = self.bounds()
        e = hi - lo
        # Aabb3::diagonal = extent().norm() with the pinned (x*x + y*y) + z*z order
        return float(np.sqrt((e[0] * e[0] + e[1] * e[1]) + e[2] * e[2]))

    def view(self) -> MfMeshView:
        """A ``mf_mesh_view`` over this mesh's arrays (kept alive by the mesh)."""
        v = MfMeshView()
        v.positions = _dptr(self.positions)
        v.n_vertices = self.vertex_count()
        v.faces = _iptr(self.faces)
        v.n_faces = self.face_count()
        v.normals = _dptr(self.normals) if self.has_normals() else ctypes.POINTER(ctypes.c_double)()
        if self.has_uvs():
            v.uvs = _dptr(self.uvs)
            v.n_uvs = int(self.uvs.shape[0])
            v.face_uvs = _iptr(self.face_uvs)
        else:
            v.uvs = ctypes.POINTER(ctypes.c_double)()
            v.n_uvs = 0 if self.uvs is None else int(self.uvs.shape[0])
            v.face_uvs = _iptr(self.face_uvs) if (self.face_uvs is not None
                                                   and self.face_uvs.shape[0] == self.faces.shape[0]) \
                else ctypes.POINTER(ctypes.c_int32)()
        return v

    def copy(self) -> "TriangleMesh":
        c = lambda a: None if a is None else a.copy()  # noqa: E731
        return TriangleMesh(self.positions.copy(), self.faces.copy(), c(self.normals), c(self.uvs),
                            c(self.face_uvs))
