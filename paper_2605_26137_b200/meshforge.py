"""Python mirror of the reference bake API, backed by the CUDA library.

Same names, argument meaning and error behaviour as the reference's C++ API
(``proj/include/meshforge/bake/gbuffer.h``, ``bake/tangent.h``,
``spatial/bvh.h``), so the parity tests read like ``tests/test_bake.cpp`` /
``tests/test_spatial.cpp``. Every call goes through the C ABI of
``libmfbake.so``; there is no CPU path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import capi
from .capi import MeshforgeError, check, default_context
from .mesh import TriangleMesh

__all__ = ["GBuffer", "rasterize_gbuffer", "transfer_normals", "dilate_seams", "bake_normal_map",
           "bake_normal_map_ex", "decode_rg16",
           "Bvh", "compute_wedge_tangents", "compute_vertex_normals", "MeshforgeError", "TriangleMesh"]


def _p(a):
    # data_as keeps a reference to `a`: temporaries stay alive through the call
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class GBuffer:
    """bake/gbuffer.h:17-30: per-texel attributes, v down the rows."""

    resolution: int
    position: np.ndarray   # (res*res, 3) f32
    normal: np.ndarray
    tangent: np.ndarray
    bitangent: np.ndarray
    valid: np.ndarray      # (res*res,) u8
    reliable: np.ndarray

    def index(self, x: int, y: int) -> int:
        return y * self.resolution + x

    def empty(self) -> bool:
        return self.valid.size == 0

    @classmethod
    def allocate(cls, res: int) -> "GBuffer":
        n = max(res, 0) ** 2
        z = lambda: np.zeros((n, 3), np.float32)  # noqa: E731
        return cls(res, z(), z(), z(), z(), np.zeros(n, np.uint8), np.zeros(n, np.uint8))


def rasterize_gbuffer(lowpoly: TriangleMesh, resolution: int, ctx=None) -> GBuffer:
    """rasterizeGBuffer (gbuffer.h:65)."""
    ctx = ctx or default_context()
    g = GBuffer.allocate(resolution)
    v = lowpoly.view()
    check(ctx.lib.mf_raster_gbuffer(ctx.h, ctypes.byref(v), int(resolution), _p(g.position), _p(g.normal),
                                    _p(g.tangent), _p(g.bitangent), _p(g.valid), _p(g.reliable)))
    return g


def transfer_normals(gbuffer: GBuffer, highpoly: TriangleMesh, bbox_diagonal: float,
                     max_distance_fraction: float = 0.01, ctx=None) -> np.ndarray:
    """transferNormals (gbuffer.h:72-73); returns an RGB8 image (res, res, 3)."""
    ctx = ctx or default_context()
    res = gbuffer.resolution if not gbuffer.empty() else 0
    out = np.zeros((max(res, 1), max(res, 1), 3), np.uint8) if res > 0 else np.zeros((0, 0, 3), np.uint8)
    v = highpoly.view()
    valid = gbuffer.valid if not gbuffer.empty() else None
    check(ctx.lib.mf_transfer_normals(ctx.h, int(res), _p(gbuffer.position), _p(gbuffer.normal),
                                      _p(gbuffer.tangent), _p(gbuffer.bitangent), _p(valid),
                                      _p(gbuffer.reliable), ctypes.byref(v), float(bbox_diagonal),
                                      float(max_distance_fraction), _p(out)))
    return out


def dilate_seams(image: np.ndarray, gbuffer: GBuffer, radius: int = 4, ctx=None) -> np.ndarray:
    """dilateSeams (gbuffer.h:79). ``image`` is (h, w, c) uint8."""
    ctx = ctx or default_context()
    img = np.ascontiguousarray(image, dtype=np.uint8)
    if img.ndim == 2:
        img = img[:, :, None]
    h, w, c = img.shape
    out = np.empty_like(img)
    check(ctx.lib.mf_dilate_seams(ctx.h, int(w), int(h), int(c), _p(img), int(gbuffer.resolution),
                                  _p(np.ascontiguousarray(gbuffer.valid, np.uint8)), int(radius), _p(out)))
    return out


def bake_normal_map(lowpoly: TriangleMesh, highpoly: TriangleMesh, resolution: int, bbox_diagonal: float,
                    max_distance_fraction: float = 0.01, radius: int = 4, debug: bool = False,
                    stats: bool = False, ctx=None, out=None):
    """dilateSeams(transferNormals(rasterizeGBuffer(lo, res), hi, diag, frac), g, radius)
    (test_bake.cpp:205-206) in one device-resident call. With ``debug`` also
    returns per-texel hit faces and pre-quantisation tangent-space vectors.
    ``out`` (optional): a caller-owned (res, res, 3) uint8 C-contiguous array
    to write into, e.g. a view of pinned host memory."""
    ctx = ctx or default_context()
    res = int(resolution)
    if out is None:
        out = np.zeros((res, res, 3), np.uint8) if res > 0 else np.zeros((0, 0, 3), np.uint8)
    elif out.shape != (res, res, 3) or out.dtype != np.uint8 or not out.flags["C_CONTIGUOUS"]:
        raise ValueError("out must be a C-contiguous (res, res, 3) uint8 array")
    face = np.zeros(res * res, np.int32) if debug and res > 0 else None
    ts = np.zeros((res * res, 3), np.float64) if debug and res > 0 else None
    st = capi.MfBakeStats()
    lv, hv = lowpoly.view(), highpoly.view()
    check(ctx.lib.mf_bake_normal_map(ctx.h, ctypes.byref(lv), ctypes.byref(hv), res, float(bbox_diagonal),
                                     float(max_distance_fraction), int(radius), _p(out), _p(face), _p(ts),
                                     ctypes.byref(st)))
    if not debug and not stats:
        return out
    result = {"rgb": out}
    if debug:
        result.update(face=face, ts=ts)
    if stats:
        result["stats"] = st.as_dict()
    return result


ATLAS_RGB8, ATLAS_RGBA8, ATLAS_RG16 = 0, 1, 2  # MF_ATLAS_* (include/mfbake.h)
_ATLAS_SHAPE = {ATLAS_RGB8: (3, np.uint8), ATLAS_RGBA8: (4, np.uint8), ATLAS_RG16: (2, np.uint16)}


def bake_normal_map_ex(lowpoly: TriangleMesh, highpoly: TriangleMesh, resolution: int, bbox_diagonal: float,
                       max_distance_fraction: float = 0.01, radius: int = 4, fmt: int = ATLAS_RGBA8,
                       stats: bool = False, ctx=None, out=None):
    """bake_normal_map with an atlas encoding (mf_bake_normal_map_ex): RGB8
    -> (res, res, 3) uint8, RGBA8 -> (res, res, 4) uint8 (alpha 255), RG16
    -> (res, res, 2) uint16 (tangent-space x, y as unorm16)."""
    ctx = ctx or default_context()
    res = int(resolution)
    ch, dt = _ATLAS_SHAPE.get(fmt, (4, np.uint8))
    if out is None:
        out = np.zeros((max(res, 0), max(res, 0), ch), dt)
    elif out.shape != (res, res, ch) or out.dtype != dt or not out.flags["C_CONTIGUOUS"]:
        raise ValueError(f"out must be a C-contiguous (res, res, {ch}) {np.dtype(dt).name} array")
    st = capi.MfBakeStats()
    lv, hv = lowpoly.view(), highpoly.view()
    check(ctx.lib.mf_bake_normal_map_ex(ctx.h, ctypes.byref(lv), ctypes.byref(hv), res, float(bbox_diagonal),
                                        float(max_distance_fraction), int(radius), int(fmt), _p(out),
                                        ctypes.byref(st)))
    if not stats:
        return out
    return {"atlas": out, "stats": st.as_dict()}


def decode_rg16(atlas: np.ndarray) -> np.ndarray:
    """RG16 atlas -> (res, res, 3) f64 tangent-space vectors (z reconstructed)."""
    xy = atlas.astype(np.float64) / 65535.0 * 2.0 - 1.0
    z = np.sqrt(np.clip(1.0 - (xy ** 2).sum(-1), 0.0, None))
    return np.concatenate([xy, z[..., None]], -1)


def compute_wedge_tangents(mesh: TriangleMesh, ctx=None) -> np.ndarray:
    """computeWedgeTangents (tangent.h:22): (F, 3, 3, 3) = [face][corner][T,B,N][xyz]."""
    ctx = ctx or default_context()
    out = np.zeros((mesh.face_count(), 3, 3, 3))
    v = mesh.view()
    check(ctx.lib.mf_wedge_tangents(ctx.h, ctypes.byref(v), _p(out)))
    return out


def compute_vertex_normals(mesh: TriangleMesh, ctx=None) -> np.ndarray:
    """computeVertexNormals (core/mesh.h:39)."""
    ctx = ctx or default_context()
    out = np.zeros((mesh.vertex_count(), 3))
    v = mesh.view()
    check(ctx.lib.mf_vertex_normals(ctx.h, ctypes.byref(v), _p(out)))
    return out


class Bvh:
    """spatial/bvh.h:30-69 on the device (an LBVH; results equal the
    reference's median-split tree because queries are tree-independent)."""

    def __init__(self, mesh: TriangleMesh, ctx=None):
        self.ctx = ctx or default_context()
        self.mesh = mesh
        self._dm = capi.DeviceMesh(self.ctx, mesh)
        h = ctypes.c_void_p()
        check(self.ctx.lib.mf_bvh_build(self.ctx.h, self._dm.h, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.mf_bvh_destroy(self.h)
            self.h = None
        if getattr(self, "_dm", None):
            self._dm.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # bulk forms -------------------------------------------------------------
    def closest_points(self, queries: np.ndarray, max_distance: float = float("inf")):
        q = np.ascontiguousarray(queries, np.float64).reshape(-1, 3)
        n = q.shape[0]
        face = np.zeros(n, np.int32)
        ds = np.zeros(n)
        pt = np.zeros((n, 3))
        bary = np.zeros((n, 3))
        check(self.ctx.lib.mf_bvh_closest_within(self.h, _p(q), n, float(max_distance), _p(face), _p(ds), _p(pt),
                                                 _p(bary)))
        return face, ds, pt, bary

    def raycasts(self, origins: np.ndarray, dirs: np.ndarray, t_min: float = 0.0, t_max: float = float("inf")):
        o = np.ascontiguousarray(origins, np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
        n = o.shape[0]
        face = np.zeros(n, np.int32)
        t, u, v = np.zeros(n), np.zeros(n), np.zeros(n)
        check(self.ctx.lib.mf_bvh_raycast_first(self.h, _p(o), _p(d), n, float(t_min), float(t_max), _p(face),
                                                _p(t), _p(u), _p(v)))
        return face, t, u, v

    # single-query forms mirroring the reference ---------------------------------
    def closest_point_within(self, q, max_distance: float):
        f, ds, pt, b = self.closest_points(np.asarray(q, np.float64)[None], max_distance)
        return SurfacePoint(int(f[0]), float(ds[0]), pt[0], b[0])

    def closest_point(self, q):
        return self.closest_point_within(q, float("inf"))

    def raycast_first(self, origin, direction, t_min: float = 0.0, t_max: float = float("inf")):
        f, t, u, v = self.raycasts(np.asarray(origin, np.float64)[None], np.asarray(direction, np.float64)[None],
                                   t_min, t_max)
        return RayHit(int(f[0]), float(t[0]), float(u[0]), float(v[0]))

    def sample_sdf(self, grid_res: int, origin, voxel_size: float, field: np.ndarray, points: np.ndarray):
        """sampleSdf (signfield/watertight.cpp:29-38) with this tree as the
        watertight mesh's: sign(trilinear field) * closest distance."""
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        fld = np.ascontiguousarray(field, np.float32).reshape(-1)
        org = np.ascontiguousarray(origin, np.float64).reshape(3)
        out = np.zeros(len(pts))
        check(self.ctx.lib.mf_sample_sdf(self.h, int(grid_res), _p(org), float(voxel_size), _p(fld), _p(pts),
                                         len(pts), _p(out)))
        return out

    def surface_band(self, resolution: int = 128, band_voxels: float = 1.0, dilate_radius: int = 2,
                     domain=None):
        """markSurfaceBand (signfield/sign_grid.cpp:23-69) on this tree's mesh:
        (labels u8 res^3 with 0 = Unknown / 1 = SurfaceBand, distance f32 res^3,
        grid dict), x fastest as SignGrid::index (sign_grid.h:27-29)."""
        n = resolution ** 3
        labels = np.zeros(n, np.uint8)
        dist = np.zeros(n, np.float32)
        grid = np.zeros(5)
        dom = None if domain is None else np.ascontiguousarray(domain, dtype=np.float64).reshape(6)
        check(self.ctx.lib.mf_surface_band(self.h, int(resolution), float(band_voxels), int(dilate_radius),
                                           _p(dom), _p(labels), _p(dist), _p(grid)))
        return labels, dist, dict(origin=grid[:3].copy(), voxel_size=float(grid[3]), truncation=float(grid[4]))

    def info(self):
        nodes, leaves, depth = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        check(self.ctx.lib.mf_bvh_info(self.h, ctypes.byref(nodes), ctypes.byref(leaves), ctypes.byref(depth)))
        return nodes.value, leaves.value, depth.value

    def export(self):
        """Nodes in the reference layout (bvh.h:32-39): boxes (N, 6), links (N, 4)
        = (left, right, first, count), plus faceOrder."""
        n, _, _ = self.info()
        boxes = np.zeros((n, 6))
        links = np.zeros((n, 4), np.int32)
        order = np.zeros(self.mesh.face_count(), np.int32)
        check(self.ctx.lib.mf_bvh_export(self.h, _p(boxes), _p(links), _p(order)))
        return boxes, links, order


@dataclass
class SurfacePoint:
    face: int = -1
    distance_squared: float = float("inf")
    point: Optional[np.ndarray] = None
    barycentric: Optional[np.ndarray] = None

    def valid(self) -> bool:
        return self.face >= 0

    def distance(self) -> float:
        return float(np.sqrt(self.distance_squared))


@dataclass
class RayHit:
    face: int = -1
    t: float = float("inf")
    u: float = 0.0
    v: float = 0.0

    def valid(self) -> bool:
        return self.face >= 0


# ---------------------------------------------------------------- ortho views
def fibonacci_cameras(count: int, half_extent: float = 0.52, ctx=None) -> np.ndarray:
    """fibonacciCameras (render/camera.cpp:38-55): count x 7 = direction xyz, up xyz, halfExtent."""
    ctx = ctx or default_context()
    cams = np.zeros((count, 7))
    check(ctx.lib.mf_fibonacci_cameras(int(count), float(half_extent), _p(cams)))
    return cams


def render_views(mesh: TriangleMesh, cameras: np.ndarray, resolution: int, vertex_normals=None,
                 backface_cull: bool = False, ctx=None):
    """renderView (render/raster.cpp:12-102) for each camera row: (face i32, depth f32,
    position f32x3, normal f32x3) per view, one pixel ray per thread through the LBVH."""
    ctx = ctx or default_context()
    cams = np.ascontiguousarray(cameras, dtype=np.float64).reshape(-1, 7)
    n = cams.shape[0]
    face = np.zeros((n, resolution, resolution), np.int32)
    depth = np.zeros((n, resolution, resolution), np.float32)
    pos = np.zeros((n, resolution, resolution, 3), np.float32)
    nrm = np.zeros((n, resolution, resolution, 3), np.float32)
    vn = None if vertex_normals is None else np.ascontiguousarray(vertex_normals, dtype=np.float64)
    v = mesh.view()
    check(ctx.lib.mf_render_views(ctx.h, ctypes.byref(v), _p(cams), n, int(resolution), _p(vn), int(backface_cull),
                                  _p(face), _p(depth), _p(pos), _p(nrm)))
    return face, depth, pos, nrm


def cast_visibility(mesh: TriangleMesh, viewpoints: int = 512, resolution: int = 1024, ctx=None):
    """castVisibility (visibility/visibility.cpp:13-59): (hits i64 per face, state u8 0 Hidden / 1 Visible)."""
    ctx = ctx or default_context()
    hits = np.zeros(mesh.face_count(), np.int64)
    state = np.zeros(mesh.face_count(), np.uint8)
    v = mesh.view()
    check(ctx.lib.mf_cast_visibility(ctx.h, ctypes.byref(v), int(viewpoints), int(resolution), _p(hits), _p(state)))
    return hits, state
