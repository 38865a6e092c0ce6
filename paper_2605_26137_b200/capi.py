"""ctypes bindings of libmfbake.so (the C ABI declared in include/mfbake.h).

The product path has no CPU fallback: if the CUDA library is missing or no
device is present, every call raises ``MfbakeUnavailable`` / ``MeshforgeError``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

from .mesh import MfMeshView, TriangleMesh

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MFB_LIB") or os.path.join(HERE, "libmfbake.so")

# include/mfbake.h status codes (1 + meshforge::ErrorCode, error.h:8-21)
ERROR_NAMES = {
    1: "EmptyMesh", 2: "InvalidGeometry", 3: "OutOfBounds", 4: "EmptySurface", 5: "AllHidden",
    6: "ChartFailure", 7: "PackOverflow", 8: "AtlasOverlap", 9: "ShapeMismatch", 10: "NothingToInpaint",
    11: "ExportMismatch", 12: "InvalidConfig", 13: "IoError",
    -1: "CudaError", -2: "OutOfMemory", -3: "BadArgument", -4: "NoDevice",
}
VALIDATION = {"EmptyMesh", "InvalidGeometry", "OutOfBounds", "InvalidConfig", "ShapeMismatch", "ExportMismatch"}


class MfbakeUnavailable(RuntimeError):
    pass


class MeshforgeError(RuntimeError):
    """Mirror of meshforge::Error (core/error.h:28-43): carries the code name."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = ERROR_NAMES.get(status, f"Status{status}")
        super().__init__(message if message.startswith(self.code) else f"{self.code}: {message}")

    def is_validation(self) -> bool:
        return self.code in VALIDATION


class MfBakeStats(ctypes.Structure):
    _fields_ = [
        ("valid_texels", ctypes.c_int64), ("queries", ctypes.c_int64), ("hits", ctypes.c_int64),
        ("bvh_nodes", ctypes.c_int32), ("bvh_depth", ctypes.c_int32),
        ("ms_upload", ctypes.c_float), ("ms_prepare", ctypes.c_float), ("ms_bvh", ctypes.c_float),
        ("ms_raster", ctypes.c_float), ("ms_transfer", ctypes.c_float), ("ms_dilate", ctypes.c_float),
        ("ms_download", ctypes.c_float), ("ms_total", ctypes.c_float),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_VP = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_I64 = ctypes.c_int64
_MV = ctypes.POINTER(MfMeshView)

# (name, restype, argtypes) for every symbol include/mfbake.h declares
SIGNATURES = [
    ("mf_version", ctypes.c_char_p, []),
    ("mf_abi_version", _I, []),
    ("mf_last_error", ctypes.c_char_p, []),
    ("mf_ctx_create", _I, [_I, _VP, ctypes.POINTER(_VP)]),
    ("mf_ctx_destroy", None, [_VP]),
    ("mf_ctx_synchronize", _I, [_VP]),
    ("mf_ctx_set_timing", _I, [_VP, _I]),
    ("mf_ctx_launch_count", _I64, [_VP]),
    ("mf_mesh_upload", _I, [_VP, _MV, ctypes.POINTER(_VP)]),
    ("mf_mesh_destroy", None, [_VP]),
    ("mf_raster_gbuffer", _I, [_VP, _MV, _I, _VP, _VP, _VP, _VP, _VP, _VP]),
    ("mf_transfer_normals", _I, [_VP, _I, _VP, _VP, _VP, _VP, _VP, _VP, _MV, _D, _D, _VP]),
    ("mf_dilate_seams", _I, [_VP, _I, _I, _I, _VP, _I, _VP, _I, _VP]),
    ("mf_bake_normal_map", _I, [_VP, _MV, _MV, _I, _D, _D, _I, _VP, _VP, _VP, ctypes.POINTER(MfBakeStats)]),
    ("mf_bake_normal_map_ex", _I, [_VP, _MV, _MV, _I, _D, _D, _I, _I, _VP, ctypes.POINTER(MfBakeStats)]),
    ("mf_bake_normal_map_dev", _I, [_VP, _VP, _VP, _I, _D, _D, _I, _I, _I, _VP, ctypes.POINTER(MfBakeStats)]),
    ("mf_bake_normal_map_dev_ex", _I, [_VP, _VP, _VP, _I, _D, _D, _I, _I, _I, _I, _VP,
                                       ctypes.POINTER(MfBakeStats)]),
    ("mf_coverage_rows", _I, [_VP, _VP, _I, _VP]),
    ("mf_bvh_build", _I, [_VP, _VP, ctypes.POINTER(_VP)]),
    ("mf_bvh_destroy", None, [_VP]),
    ("mf_bvh_set_stream", ctypes.c_int, [_VP, _VP]),
    ("mf_bvh_info", _I, [_VP, _VP, _VP, _VP]),
    ("mf_bvh_export", _I, [_VP, _VP, _VP, _VP]),
    ("mf_bvh_closest_within", _I, [_VP, _VP, _I64, _D, _VP, _VP, _VP, _VP]),
    ("mf_bvh_closest_within_dev", _I, [_VP, _VP, _I64, _D, _VP, _VP, _VP, _VP]),
    ("mf_bvh_raycast_first", _I, [_VP, _VP, _VP, _I64, _D, _D, _VP, _VP, _VP, _VP]),
    ("mf_bvh_raycast_first_dev", _I, [_VP, _VP, _VP, _I64, _D, _D, _VP, _VP, _VP, _VP]),
    ("mf_ipc_export", _I, [_VP, _VP, ctypes.POINTER(ctypes.c_uint64)]),
    ("mf_ipc_open", _I, [_VP, _VP, ctypes.c_uint64, ctypes.POINTER(_VP)]),
    ("mf_ipc_close", _I, [_VP, _VP]),
    ("mf_bake_normal_map_dev_publish", _I, [_VP, _VP, _VP, _I, _D, _D, _I, _I, _I, _VP, _I,
                                            ctypes.POINTER(MfBakeStats)]),
    ("mf_sample_sdf", _I, [_VP, _I, _VP, _D, _VP, _VP, _I64, _VP]),
    ("mf_sample_sdf_dev", _I, [_VP, _I, _VP, _D, _VP, _VP, _I64, _VP]),
    ("mf_surface_band", _I, [_VP, _I, _D, _I, _VP, _VP, _VP, _VP]),
    ("mf_surface_band_dev", _I, [_VP, _I, _D, _I, _VP, _VP, _VP, _VP]),
    ("mf_fibonacci_cameras", _I, [_I, _D, _VP]),
    ("mf_render_views", _I, [_VP, _MV, _VP, _I, _I, _VP, _I, _VP, _VP, _VP, _VP]),
    ("mf_cast_visibility", _I, [_VP, _MV, _I, _I, _VP, _VP]),
    ("mf_closest_point_brute", _I, [_VP, _MV, _VP, _I64, _VP, _VP, _VP, _VP]),
    ("mf_raycast_first_brute", _I, [_VP, _MV, _VP, _VP, _I64, _D, _D, _VP, _VP, _VP, _VP]),
    ("mf_fuse_options_default", None, [_VP]),
    ("mf_mip_chain_floats", _I64, [_I, _I, _I, _I, _VP]),
    ("mf_edge_mask", _I, [_VP, _I, _I, _VP, _VP, _D, _D, _VP]),
    ("mf_build_mips", _I, [_VP, _I, _I, _I, _VP, _I, ctypes.c_float, _VP, _VP]),
    ("mf_backproject_view", _I, [_VP, _I, _VP, _VP, _VP, _I, _I, _I, _VP, _VP, _VP, _VP]),
    ("mf_incidence_map", _I, [_VP, _I, _VP, _VP, _VP, _VP, _I, _VP, _D, _D, _VP]),
    ("mf_blend_views", _I, [_VP, _I, _I, _I, _I, _VP, _VP, _VP, _VP, _D, _D, _VP, _VP]),
    ("mf_fuse_views", _I, [_VP, _I, _VP, _VP, _VP, _I, _VP, _I, _VP, _VP, _VP, _I, _VP, _VP, _D, _VP, _VP, _VP]),
    ("mf_fuse_views_dev", _I, [_VP, _I, _VP, _VP, _VP, _I, _VP, _I, _VP, _VP, _VP, _I, _VP, _VP, _D, _VP, _VP,
                               _VP]),
    ("mf_raster_gbuffer_dev", _I, [_VP, _VP, _I, _VP, _VP, _VP, _VP, _VP, _VP]),
    ("mf_wedge_tangents", _I, [_VP, _MV, _VP]),
    ("mf_vertex_normals", _I, [_VP, _MV, _VP]),
]

_lib: Optional[ctypes.CDLL] = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libmfbake.so and bind every declared symbol (raises if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise MfbakeUnavailable(f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def check(status: int):
    if status != 0:
        raise MeshforgeError(status, load().mf_last_error().decode(errors="replace"))


class Context:
    """An mf_ctx: one device + stream (+ a side stream) and its scratch."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        lib = load()
        h = ctypes.c_void_p()
        check(lib.mf_ctx_create(device, ctypes.c_void_p(stream) if stream else None, ctypes.byref(h)))
        self.h = h
        self.lib = lib

    def close(self):
        if getattr(self, "h", None):
            self.lib.mf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        check(self.lib.mf_ctx_synchronize(self.h))

    def set_timing(self, on: bool = True):
        check(self.lib.mf_ctx_set_timing(self.h, 1 if on else 0))

    @property
    def launches(self) -> int:
        return int(self.lib.mf_ctx_launch_count(self.h))


class DeviceMesh:
    """A device-resident mf_mesh (validated at upload)."""

    def __init__(self, ctx: Context, mesh: TriangleMesh):
        self.ctx = ctx
        self.mesh = mesh
        v = mesh.view()
        h = ctypes.c_void_p()
        check(ctx.lib.mf_mesh_upload(ctx.h, ctypes.byref(v), ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.mf_mesh_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx
