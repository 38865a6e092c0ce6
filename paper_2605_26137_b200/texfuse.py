"""Texture fusion on the device: Python mirror of
proj/include/meshforge/texfuse/fuse.h and mips.h over the C ABI
(include/mfbake.h, texfuse section; kernels in csrc/texfuse.cu).

Images are numpy arrays in the reference layout (ImageF: row-major,
interleaved channels): a view image is (res, res, channels) f32, a G-buffer is
mesh.GBuffer (rasterize_gbuffer). A camera is the 7-vector (direction xyz,
up xyz, halfExtent) of OrthoCamera (render/camera.h:12-38); the view
resolution is passed beside it.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

import numpy as np

from . import capi
from .capi import check, default_context

__all__ = ["FuseOptions", "edge_mask", "build_mips", "backproject_view", "incidence_map", "blend_views",
           "fuse_views", "standard_view_priors", "standard_cameras"]


class FuseOptions(ctypes.Structure):
    """mf_fuse_options: FuseOptions + BlendOptions (fuse.h:83-86, 122-130)."""
    _fields_ = [("edge_threshold", ctypes.c_double), ("depth_tolerance", ctypes.c_double),
                ("mip_levels", ctypes.c_int32), ("sharpen_strength", ctypes.c_float),
                ("alpha", ctypes.c_double), ("epsilon", ctypes.c_double)]

    @classmethod
    def defaults(cls) -> "FuseOptions":
        o = cls()
        capi.load().mf_fuse_options_default(ctypes.byref(o))
        return o


def _p(a):
    # data_as keeps a reference to the array (callers also bind their arrays
    # to locals for the duration of the call)
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, np.float32)


def standard_view_priors() -> List[float]:
    """standardViewPriors (fuse.cpp:282-284)."""
    return [1.0, 0.1, 0.01, 0.001, 1.0, 0.001, 0.01, 0.1, 0.3, 0.3]


def standard_cameras(half_extent: float = 0.52) -> np.ndarray:
    """standardCameras (render/camera.cpp:7-27) as (10, 7) camera vectors."""
    s2 = np.sqrt(0.5)
    cos_a = [1, s2, 0, -s2, -1, -s2, 0, s2]
    sin_a = [0, s2, 1, s2, 0, -s2, -1, -s2]
    cams = np.zeros((10, 7))
    for k in range(8):
        cams[k, :3] = (-cos_a[k], -sin_a[k], 0.0)
        cams[k, 3:6] = (0, 0, 1)
    cams[8, :3], cams[8, 3:6] = (0, 0, -1), (0, 1, 0)
    cams[9, :3], cams[9, 3:6] = (0, 0, 1), (0, 1, 0)
    cams[:, 6] = half_extent
    return cams


def edge_mask(position: np.ndarray, face: np.ndarray, bbox_diagonal: float, threshold: float = 0.02,
              ctx=None) -> np.ndarray:
    """edgeMask (fuse.cpp:66-101): (h, w) u8, 1 = do not sample."""
    ctx = ctx or default_context()
    face = np.ascontiguousarray(face, np.int32)
    position = _f32(position)
    h, w = face.shape
    mask = np.zeros((h, w), np.uint8)
    check(ctx.lib.mf_edge_mask(ctx.h, w, h, _p(position), _p(face), float(bbox_diagonal), float(threshold),
                               _p(mask)))
    return mask


def _chain_shapes(w: int, h: int, levels: int):
    dims = [(w, h)]
    while len(dims) < levels and dims[-1] != (1, 1):
        pw, ph = dims[-1]
        dims.append((max(1, (pw + 1) // 2), max(1, (ph + 1) // 2)))
    return dims


def build_mips(base: np.ndarray, levels: int = 6, sharpen: float = 0.2, ctx=None) -> List[np.ndarray]:
    """buildMips (mips.cpp:96-112): the chain as a list of (h_l, w_l, c) arrays."""
    ctx = ctx or default_context()
    base = _f32(base)
    h, w, c = base.shape
    n = ctypes.c_int(0)
    total = int(ctx.lib.mf_mip_chain_floats(w, h, c, int(levels), ctypes.byref(n)))
    flat = np.zeros(max(total, 1), np.float32)
    check(ctx.lib.mf_build_mips(ctx.h, w, h, c, _p(base), int(levels), ctypes.c_float(sharpen), _p(flat),
                                ctypes.byref(n)))
    out, o = [], 0
    for (lw, lh) in _chain_shapes(w, h, n.value):
        out.append(flat[o:o + lw * lh * c].reshape(lh, lw, c))
        o += lw * lh * c
    return out


def _flat_chain(mips: Sequence[np.ndarray]) -> np.ndarray:
    return np.concatenate([_f32(m).reshape(-1) for m in mips])


def backproject_view(gbuffer, camera: np.ndarray, view_res: int, mips: Sequence[np.ndarray], mask: np.ndarray,
                     ctx=None):
    """backprojectView (fuse.cpp:103-186) -> (color (res, res, c) f32, sampled (res, res) u8)."""
    ctx = ctx or default_context()
    if not mips or mips[0].shape[0] < 1:
        raise capi.MeshforgeError(12, "view mip chain is empty")  # InvalidConfig
    c = mips[0].shape[2]
    if mips[0].shape[:2] != (view_res, view_res):
        raise capi.MeshforgeError(9, "view image does not match the camera")
    if np.asarray(mask).size != view_res * view_res:
        raise capi.MeshforgeError(9, "edge mask does not match the view")
    n = gbuffer.resolution
    color = np.zeros((max(n, 0), max(n, 0), c), np.float32)
    sampled = np.zeros((max(n, 0), max(n, 0)), np.uint8)
    pos, valid = _f32(gbuffer.position), (np.ascontiguousarray(gbuffer.valid, np.uint8) if n > 0 else None)
    cam, chain, mask = np.ascontiguousarray(camera, np.float64), _flat_chain(mips), np.ascontiguousarray(mask, np.uint8)
    check(ctx.lib.mf_backproject_view(ctx.h, n, _p(pos), _p(valid), _p(cam), int(view_res), c, len(mips), _p(chain),
                                      _p(mask), _p(color), _p(sampled)))
    return color, sampled


def incidence_map(gbuffer, camera: np.ndarray, view_res: int, depth: np.ndarray, bbox_diagonal: float,
                  depth_tolerance: float = 0.005, ctx=None) -> np.ndarray:
    """incidenceMap (fuse.cpp:188-221) -> (res, res) f32."""
    ctx = ctx or default_context()
    if np.asarray(depth).shape[:2] != (view_res, view_res):
        raise capi.MeshforgeError(9, "depth buffer does not match the camera")
    n = gbuffer.resolution
    out = np.zeros((max(n, 0), max(n, 0)), np.float32)
    pos, nrm = _f32(gbuffer.position), _f32(gbuffer.normal)
    valid = np.ascontiguousarray(gbuffer.valid, np.uint8) if n > 0 else None
    cam, depth = np.ascontiguousarray(camera, np.float64), _f32(depth)
    check(ctx.lib.mf_incidence_map(ctx.h, n, _p(pos), _p(nrm), _p(valid), _p(cam), int(view_res), _p(depth),
                                   float(bbox_diagonal), float(depth_tolerance), _p(out)))
    return out


def blend_views(colors: Sequence[np.ndarray], sampled: Sequence[np.ndarray], incidence: Sequence[np.ndarray],
                priors: Sequence[float], alpha: float = 4.0, epsilon: float = 1e-8, ctx=None):
    """blendViews (fuse.cpp:223-280) -> (color (h, w, c) f32, filled (h, w) u8)."""
    ctx = ctx or default_context()
    k = len(colors)
    if k == 0:
        check(ctx.lib.mf_blend_views(ctx.h, 0, 0, 0, 0, None, None, None, None, float(alpha), float(epsilon), None,
                                     None))
    if len(incidence) != k or len(priors) != k:
        raise capi.MeshforgeError(12, "views, incidence maps and priors must pair up")
    h, w, c = colors[0].shape
    for i in range(k):
        if colors[i].shape != (h, w, c) or np.asarray(sampled[i]).size != h * w:
            raise capi.MeshforgeError(9, "partial atlases disagree on resolution")
        if np.asarray(incidence[i]).size != h * w:
            raise capi.MeshforgeError(9, "incidence maps disagree on resolution")
    out = np.zeros((h, w, c), np.float32)
    filled = np.zeros((h, w), np.uint8)
    cols, samp, inc = _f32(np.stack(colors)), np.ascontiguousarray(np.stack(sampled), np.uint8), \
        _f32(np.stack(incidence))
    pri = np.ascontiguousarray(priors, np.float64)
    check(ctx.lib.mf_blend_views(ctx.h, k, w, h, c, _p(cols), _p(samp), _p(inc), _p(pri), float(alpha),
                                 float(epsilon), _p(out), _p(filled)))
    return out, filled


def fuse_views(gbuffer, cameras: np.ndarray, view_res: int, view_position: np.ndarray, view_face: np.ndarray,
               view_depth: np.ndarray, colors: np.ndarray, priors: Sequence[float], bbox_diagonal: float,
               options: Optional[FuseOptions] = None, ctx=None):
    """fuseViews (fuse.cpp:292-326) up to the blend, device-resident in one
    call: views stacked as (k, res, res, ...) arrays. -> (color, filled)."""
    ctx = ctx or default_context()
    cams = np.ascontiguousarray(cameras, np.float64).reshape(-1, 7)
    k = cams.shape[0]
    colors = _f32(colors)
    c = colors.shape[-1]
    n = gbuffer.resolution
    out = np.zeros((max(n, 0), max(n, 0), c), np.float32)
    filled = np.zeros((max(n, 0), max(n, 0)), np.uint8)
    pos, nrm = _f32(gbuffer.position), _f32(gbuffer.normal)
    valid = np.ascontiguousarray(gbuffer.valid, np.uint8) if n > 0 else None
    vpos, vface, vdepth = _f32(view_position), np.ascontiguousarray(view_face, np.int32), _f32(view_depth)
    pri = np.ascontiguousarray(priors, np.float64)
    check(ctx.lib.mf_fuse_views(ctx.h, n, _p(pos), _p(nrm), _p(valid), k, _p(cams), int(view_res), _p(vpos),
                                _p(vface), _p(vdepth), c, _p(colors), _p(pri), float(bbox_diagonal),
                                None if options is None else ctypes.byref(options), _p(out), _p(filled)))
    return out, filled
