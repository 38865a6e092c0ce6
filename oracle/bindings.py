"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

Both libraries take the ``mf_mesh_view`` of include/mfbake.h and return the
same status codes (0 ok, 1 + meshforge ErrorCode, negative runtime errors).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from paper_2605_26137_b200.mesh import MfMeshView, TriangleMesh

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libmfref.so")

_VP = ctypes.c_void_p
_P = ctypes.POINTER


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_VP)


@dataclass
class GBufferArrays:
    res: int
    position: np.ndarray
    normal: np.ndarray
    tangent: np.ndarray
    bitangent: np.ndarray
    valid: np.ndarray
    reliable: np.ndarray

    @classmethod
    def empty(cls, res: int) -> "GBufferArrays":
        n = res * res
        z = lambda: np.zeros((n, 3), np.float32)  # noqa: E731
        return cls(res, z(), z(), z(), z(), np.zeros(n, np.uint8), np.zeros(n, np.uint8))

    def ptrs(self):
        return [_ptr(self.position), _ptr(self.normal), _ptr(self.tangent), _ptr(self.bitangent),
                _ptr(self.valid), _ptr(self.reliable)]


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = ctypes.CDLL(path)
        self.path = path
        err = getattr(self.lib, self.prefix + "last_error")
        err.restype = ctypes.c_char_p
        self._err = err

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self._err().decode(errors="replace"))

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)


class Port(_Lib):
    """The plain-C restatement (oracle/mf_oracle.c)."""

    prefix = "orc_"

    def raster_gbuffer(self, lo: TriangleMesh, res: int) -> GBufferArrays:
        g = GBufferArrays.empty(max(res, 0))
        v = lo.view()
        self._check(self.fn("raster_gbuffer")(ctypes.byref(v), ctypes.c_int(res), *g.ptrs()))
        return g

    def transfer_normals(self, g: GBufferArrays, hi: TriangleMesh, diag: float, frac: float = 0.01,
                         debug: bool = False, threads: int = 0):
        n = g.res * g.res
        rgb = np.zeros((n, 3), np.uint8)
        face = np.zeros(n, np.int32) if debug else None
        ts = np.zeros((n, 3), np.float64) if debug else None
        v = hi.view()
        self._check(self.fn("transfer_normals")(
            ctypes.c_int(g.res), *g.ptrs(), ctypes.byref(v), ctypes.c_double(diag),
            ctypes.c_double(frac), _ptr(rgb), _ptr(face), _ptr(ts), ctypes.c_int(threads)))
        return (rgb, face, ts) if debug else rgb

    def dilate_seams(self, rgb: np.ndarray, width: int, height: int, channels: int,
                     gres: int, valid: np.ndarray, radius: int) -> np.ndarray:
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        out = np.zeros_like(rgb)
        valid = np.ascontiguousarray(valid, dtype=np.uint8)
        self._check(self.fn("dilate_seams")(ctypes.c_int(width), ctypes.c_int(height),
                                            ctypes.c_int(channels), _ptr(rgb), ctypes.c_int(gres),
                                            _ptr(valid), ctypes.c_int(radius), _ptr(out)))
        return out

    def bake(self, lo: TriangleMesh, hi: TriangleMesh, res: int, diag: float, frac: float = 0.01,
             radius: int = 4, threads: int = 0, debug: bool = False):
        n = res * res
        rgb = np.zeros((n, 3), np.uint8)
        raw = np.zeros((n, 3), np.uint8)
        face = np.zeros(n, np.int32) if debug else None
        ts = np.zeros((n, 3), np.float64) if debug else None
        nv, nq = ctypes.c_int64(0), ctypes.c_int64(0)
        lv, hv = lo.view(), hi.view()
        self._check(self.fn("bake")(ctypes.byref(lv), ctypes.byref(hv), ctypes.c_int(res),
                                    ctypes.c_double(diag), ctypes.c_double(frac), ctypes.c_int(radius),
                                    _ptr(rgb), _ptr(raw), _ptr(face), _ptr(ts), ctypes.c_int(threads),
                                    ctypes.byref(nv), ctypes.byref(nq)))
        return dict(rgb=rgb, rgb_raw=raw, face=face, ts=ts, n_valid=nv.value, n_queries=nq.value)

    def vertex_normals(self, m: TriangleMesh) -> np.ndarray:
        out = np.zeros((m.vertex_count(), 3))
        v = m.view()
        self._check(self.fn("vertex_normals")(ctypes.byref(v), _ptr(out)))
        return out

    def wedge_tangents(self, m: TriangleMesh) -> np.ndarray:
        out = np.zeros((m.face_count(), 3, 3, 3))
        v = m.view()
        self._check(self.fn("wedge_tangents")(ctypes.byref(v), _ptr(out)))
        return out

    def reliable_faces(self, m: TriangleMesh) -> np.ndarray:
        out = np.zeros(m.face_count(), np.uint8)
        v = m.view()
        self._check(self.fn("reliable_faces")(ctypes.byref(v), _ptr(out)))
        return out

    def closest_within(self, m: TriangleMesh, q: np.ndarray, max_dist: float = float("inf"),
                       brute: bool = False, threads: int = 0):
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
        n = q.shape[0]
        face = np.zeros(n, np.int32)
        ds = np.zeros(n)
        pt = np.zeros((n, 3))
        bary = np.zeros((n, 3))
        v = m.view()
        self._check(self.fn("closest_within")(ctypes.byref(v), _ptr(q), ctypes.c_int64(n),
                                              ctypes.c_double(max_dist), ctypes.c_int(int(brute)),
                                              ctypes.c_int(threads), _ptr(face), _ptr(ds), _ptr(pt),
                                              _ptr(bary)))
        return face, ds, pt, bary

    def fibonacci_cameras(self, count: int, half_extent: float, res: int = 0) -> np.ndarray:
        cams = np.zeros((count, 7))
        self.fn("fibonacci_cameras")(ctypes.c_int(count), ctypes.c_double(half_extent), _ptr(cams))
        return cams

    def render_views(self, m: TriangleMesh, cams: np.ndarray, res: int, vn=None, cull: bool = False):
        cams = np.ascontiguousarray(cams, dtype=np.float64).reshape(-1, 7)
        nvw = cams.shape[0]
        face = np.zeros((nvw, res, res), np.int32)
        depth = np.zeros((nvw, res, res), np.float32)
        pos = np.zeros((nvw, res, res, 3), np.float32)
        nrm = np.zeros((nvw, res, res, 3), np.float32)
        vn = None if vn is None else np.ascontiguousarray(vn, dtype=np.float64)
        v = m.view()
        self._check(self.fn("render_views")(ctypes.byref(v), _ptr(cams), ctypes.c_int(nvw), ctypes.c_int(res),
                                            _ptr(vn), ctypes.c_int(int(cull)), _ptr(face), _ptr(depth), _ptr(pos),
                                            _ptr(nrm)))
        return face, depth, pos, nrm

    def cast_visibility(self, m: TriangleMesh, viewpoints: int, res: int) -> np.ndarray:
        hits = np.zeros(m.face_count(), np.int64)
        v = m.view()
        self._check(self.fn("cast_visibility")(ctypes.byref(v), ctypes.c_int(viewpoints), ctypes.c_int(res),
                                               _ptr(hits)))
        return hits

    def surface_band(self, m: TriangleMesh, res: int, band_voxels: float = 1.0, dilate: int = 2,
                     domain=None, threads: int = 0):
        n = res ** 3
        labels, dist, grid = np.zeros(n, np.uint8), np.zeros(n, np.float32), np.zeros(5)
        dom = None if domain is None else np.ascontiguousarray(domain, dtype=np.float64).reshape(6)
        v = m.view()
        self._check(self.fn("surface_band")(ctypes.byref(v), ctypes.c_int(res), ctypes.c_double(band_voxels),
                                            ctypes.c_int(dilate), _ptr(dom), ctypes.c_int(threads),
                                            _ptr(labels), _ptr(dist), _ptr(grid)))
        return labels, dist, grid

    def raycast_first(self, m: TriangleMesh, o: np.ndarray, d: np.ndarray, tmin: float = 0.0,
                      tmax: float = float("inf"), brute: bool = False, threads: int = 0):
        o = np.ascontiguousarray(o, dtype=np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1, 3)
        n = o.shape[0]
        face = np.zeros(n, np.int32)
        t, u, vv = np.zeros(n), np.zeros(n), np.zeros(n)
        v = m.view()
        self._check(self.fn("raycast_first")(ctypes.byref(v), _ptr(o), _ptr(d), ctypes.c_int64(n),
                                             ctypes.c_double(tmin), ctypes.c_double(tmax),
                                             ctypes.c_int(int(brute)), ctypes.c_int(threads), _ptr(face),
                                             _ptr(t), _ptr(u), _ptr(vv)))
        return face, t, u, vv


class Ref(_Lib):
    """The reference's own code (oracle/_ref/libmfref.so)."""

    prefix = "ref_"

    def hardware_threads(self) -> int:
        return int(self.fn("hardware_threads")())

    def raster_gbuffer(self, lo: TriangleMesh, res: int) -> GBufferArrays:
        g = GBufferArrays.empty(max(res, 0))
        v = lo.view()
        self._check(self.fn("raster_gbuffer")(ctypes.byref(v), ctypes.c_int(res), *g.ptrs()))
        return g

    def transfer_normals(self, g: GBufferArrays, hi: TriangleMesh, diag: float, frac: float = 0.01):
        rgb = np.zeros((g.res * g.res, 3), np.uint8)
        v = hi.view()
        self._check(self.fn("transfer_normals")(ctypes.c_int(g.res), *g.ptrs(), ctypes.byref(v),
                                                ctypes.c_double(diag), ctypes.c_double(frac), _ptr(rgb)))
        return rgb

    def dilate_seams(self, rgb, width, height, channels, gres, valid, radius):
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        out = np.zeros_like(rgb)
        valid = np.ascontiguousarray(valid, dtype=np.uint8)
        self._check(self.fn("dilate_seams")(ctypes.c_int(width), ctypes.c_int(height),
                                            ctypes.c_int(channels), _ptr(rgb), ctypes.c_int(gres),
                                            _ptr(valid), ctypes.c_int(radius), _ptr(out)))
        return out

    def bake(self, lo: TriangleMesh, hi: TriangleMesh, res: int, diag: float, frac: float = 0.01,
             radius: int = 4, debug: bool = False, time_bvh: bool = False):
        n = res * res
        rgb = np.zeros((n, 3), np.uint8)
        raw = np.zeros((n, 3), np.uint8)
        face = np.zeros(n, np.int32) if debug else None
        ts = np.zeros((n, 3), np.float64) if debug else None
        times = np.zeros(5)
        counters = np.zeros(4) if debug else None
        lv, hv = lo.view(), hi.view()
        self._check(self.fn("bake")(ctypes.byref(lv), ctypes.byref(hv), ctypes.c_int(res),
                                    ctypes.c_double(diag), ctypes.c_double(frac), ctypes.c_int(radius),
                                    _ptr(rgb), _ptr(raw), _ptr(face), _ptr(ts), _ptr(times),
                                    _ptr(counters), ctypes.c_int(int(time_bvh))))
        out = dict(rgb=rgb, rgb_raw=raw, face=face, ts=ts,
                   times=dict(raster=times[0], bvh=times[1], transfer=times[2], dilate=times[3],
                              total=times[4]))
        if counters is not None:
            out.update(n_valid=int(counters[0]), n_queries=int(counters[1]), n_node=float(counters[2]),
                       n_tri=float(counters[3]))
        return out

    def sampled_counters(self, lo: TriangleMesh, hi: TriangleMesh, res: int, diag: float, frac: float,
                         stride: int):
        """Best-first traversal counters on every `stride`-th query (ref_harness.cpp)."""
        c = np.zeros(5)
        lv, hv = lo.view(), hi.view()
        self._check(self.fn("sampled_counters")(ctypes.byref(lv), ctypes.byref(hv), ctypes.c_int(res),
                                                ctypes.c_double(diag), ctypes.c_double(frac),
                                                ctypes.c_int(stride), _ptr(c)))
        return dict(n_valid=int(c[0]), n_queries=int(c[1]), sampled=int(c[2]), n_node=float(c[3]),
                    n_tri=float(c[4]), stride=stride)

    def bvh_build_time(self, m: TriangleMesh):
        s, nodes = ctypes.c_double(0), ctypes.c_int(0)
        v = m.view()
        self._check(self.fn("bvh_build_time")(ctypes.byref(v), ctypes.byref(s), ctypes.byref(nodes)))
        return s.value, nodes.value

    def closest_within(self, m: TriangleMesh, q, max_dist=float("inf"), brute=False):
        q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
        n = q.shape[0]
        face, ds, pt, bary = np.zeros(n, np.int32), np.zeros(n), np.zeros((n, 3)), np.zeros((n, 3))
        v = m.view()
        self._check(self.fn("closest_within")(ctypes.byref(v), _ptr(q), ctypes.c_int64(n),
                                              ctypes.c_double(max_dist), ctypes.c_int(int(brute)),
                                              _ptr(face), _ptr(ds), _ptr(pt), _ptr(bary)))
        return face, ds, pt, bary

    def fibonacci_cameras(self, count: int, half_extent: float, res: int = 0) -> np.ndarray:
        cams = np.zeros((count, 7))
        self.fn("fibonacci_cameras")(ctypes.c_int(count), ctypes.c_int(res), ctypes.c_double(half_extent),
                                     _ptr(cams))
        return cams

    def render_views(self, m: TriangleMesh, cams: np.ndarray, res: int, vn=None, cull: bool = False):
        cams = np.ascontiguousarray(cams, dtype=np.float64).reshape(-1, 7)
        nvw = cams.shape[0]
        face = np.zeros((nvw, res, res), np.int32)
        depth = np.zeros((nvw, res, res), np.float32)
        pos = np.zeros((nvw, res, res, 3), np.float32)
        nrm = np.zeros((nvw, res, res, 3), np.float32)
        vn = None if vn is None else np.ascontiguousarray(vn, dtype=np.float64)
        v = m.view()
        self._check(self.fn("render_views")(ctypes.byref(v), _ptr(cams), ctypes.c_int(nvw), ctypes.c_int(res),
                                            _ptr(vn), ctypes.c_int(int(cull)), _ptr(face), _ptr(depth), _ptr(pos),
                                            _ptr(nrm)))
        return face, depth, pos, nrm

    def cast_visibility(self, m: TriangleMesh, viewpoints: int, res: int) -> np.ndarray:
        hits = np.zeros(m.face_count(), np.int64)
        v = m.view()
        self._check(self.fn("cast_visibility")(ctypes.byref(v), ctypes.c_int(viewpoints), ctypes.c_int(res),
                                               _ptr(hits)))
        return hits

    def surface_band(self, m: TriangleMesh, res: int, band_voxels: float = 1.0, dilate: int = 2, domain=None):
        n = res ** 3
        labels, dist, grid = np.zeros(n, np.uint8), np.zeros(n, np.float32), np.zeros(5)
        dom = None if domain is None else np.ascontiguousarray(domain, dtype=np.float64).reshape(6)
        v = m.view()
        self._check(self.fn("surface_band")(ctypes.byref(v), ctypes.c_int(res), ctypes.c_double(band_voxels),
                                            ctypes.c_int(dilate), _ptr(dom), _ptr(labels), _ptr(dist), _ptr(grid)))
        return labels, dist, grid

    # ---- texfuse (src/texfuse/fuse.cpp, mips.cpp; ref_harness.cpp) ----
    def footprint(self, jac):
        """footprintFromJacobian: jac = [[j00, j01], [j10, j11]] -> dict."""
        j = np.asarray(jac, np.float64).reshape(2, 2)
        jc = np.ascontiguousarray(j.T).reshape(4)  # column-major
        out = np.zeros(7)
        self.fn("footprint")(_ptr(jc), _ptr(out))
        return dict(axis=out[0:2].copy(), major=out[2], minor=out[3], mip=out[4], taps=int(out[5]))

    def edge_mask(self, pos, face, diag: float, threshold: float = 0.02):
        face = np.ascontiguousarray(face, np.int32)
        h, w = face.shape
        pos = np.ascontiguousarray(pos, np.float32)
        mask = np.zeros((h, w), np.uint8)
        self._check(self.fn("edge_mask")(ctypes.c_int(w), ctypes.c_int(h), _ptr(pos), _ptr(face),
                                         ctypes.c_double(diag), ctypes.c_double(threshold), _ptr(mask)))
        return mask

    def build_mips(self, base, levels: int = 6, sharpen: float = 0.2):
        base = np.ascontiguousarray(base, np.float32)
        h, w, c = base.shape
        total, dims, ww, hh = 0, [], w, h
        for l in range(levels):
            if l and dims[-1] == (1, 1):
                break
            if l:
                ww, hh = max(1, (ww + 1) // 2), max(1, (hh + 1) // 2)
            dims.append((ww, hh))
            total += ww * hh * c
        out = np.zeros(total, np.float32)
        n = ctypes.c_int(0)
        self._check(self.fn("build_mips")(ctypes.c_int(w), ctypes.c_int(h), ctypes.c_int(c), _ptr(base),
                                          ctypes.c_int(levels), ctypes.c_float(sharpen), _ptr(out), ctypes.byref(n)))
        return out, n.value

    def backproject_view(self, gpos, gvalid, gres: int, cam7, view_res: int, channels: int, n_mips: int, mips, mask):
        color = np.zeros((gres * gres, channels), np.float32)
        sampled = np.zeros(gres * gres, np.uint8)
        self._check(self.fn("backproject_view")(
            ctypes.c_int(gres), _ptr(np.ascontiguousarray(gpos, np.float32)),
            _ptr(np.ascontiguousarray(gvalid, np.uint8)), _ptr(np.ascontiguousarray(cam7, np.float64)),
            ctypes.c_int(view_res), ctypes.c_int(channels), ctypes.c_int(n_mips),
            _ptr(np.ascontiguousarray(mips, np.float32)), _ptr(np.ascontiguousarray(mask, np.uint8)),
            _ptr(color), _ptr(sampled)))
        return color, sampled

    def incidence_map(self, gpos, gnrm, gvalid, gres: int, cam7, view_res: int, depth, diag: float,
                      tol: float = 0.005):
        out = np.zeros(gres * gres, np.float32)
        self._check(self.fn("incidence_map")(
            ctypes.c_int(gres), _ptr(np.ascontiguousarray(gpos, np.float32)),
            _ptr(np.ascontiguousarray(gnrm, np.float32)), _ptr(np.ascontiguousarray(gvalid, np.uint8)),
            _ptr(np.ascontiguousarray(cam7, np.float64)), ctypes.c_int(view_res),
            _ptr(np.ascontiguousarray(depth, np.float32)), ctypes.c_double(diag), ctypes.c_double(tol), _ptr(out)))
        return out

    def blend_views(self, colors, sampled, inc, priors, alpha: float = 4.0, eps: float = 1e-8):
        colors = np.ascontiguousarray(colors, np.float32)
        k, n, c = colors.shape
        w = int(round(np.sqrt(n)))
        out = np.zeros((n, c), np.float32)
        filled = np.zeros(n, np.uint8)
        self._check(self.fn("blend_views")(
            ctypes.c_int(k), ctypes.c_int(w), ctypes.c_int(n // w), ctypes.c_int(c), _ptr(colors),
            _ptr(np.ascontiguousarray(sampled, np.uint8)), _ptr(np.ascontiguousarray(inc, np.float32)),
            _ptr(np.ascontiguousarray(priors, np.float64)), ctypes.c_double(alpha), ctypes.c_double(eps),
            _ptr(out), _ptr(filled)))
        return out, filled

    def sample_sdf(self, m: TriangleMesh, res: int, origin, voxel: float, field, pts):
        """sampleSdf (signfield/watertight.cpp:29-38)."""
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        out = np.zeros(len(pts))
        v = m.view()
        self._check(self.fn("sample_sdf")(ctypes.byref(v), ctypes.c_int(res),
                                          _ptr(np.ascontiguousarray(origin, np.float64)), ctypes.c_double(voxel),
                                          _ptr(np.ascontiguousarray(field, np.float32)), _ptr(pts),
                                          ctypes.c_int64(len(pts)), _ptr(out)))
        return out

    def standard_cameras(self, half_extent: float = 0.52) -> np.ndarray:
        cams = np.zeros((10, 7))
        self.fn("standard_cameras")(ctypes.c_double(half_extent), _ptr(cams))
        return cams

    def raycast_first(self, m: TriangleMesh, o, d, tmin=0.0, tmax=float("inf"), brute=False):
        o = np.ascontiguousarray(o, dtype=np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1, 3)
        n = o.shape[0]
        face, t, u, vv = np.zeros(n, np.int32), np.zeros(n), np.zeros(n), np.zeros(n)
        v = m.view()
        self._check(self.fn("raycast_first")(ctypes.byref(v), _ptr(o), _ptr(d), ctypes.c_int64(n),
                                             ctypes.c_double(tmin), ctypes.c_double(tmax),
                                             ctypes.c_int(int(brute)), _ptr(face), _ptr(t), _ptr(u),
                                             _ptr(vv)))
        return face, t, u, vv

    def bvh_export(self, m: TriangleMesh):
        v = m.view()
        nn = ctypes.c_int(0)
        self._check(self.fn("bvh_export")(ctypes.byref(v), ctypes.byref(nn), None, None, None))
        boxes = np.zeros((nn.value, 6))
        links = np.zeros((nn.value, 4), np.int32)
        order = np.zeros(m.face_count(), np.int32)
        self._check(self.fn("bvh_export")(ctypes.byref(v), ctypes.byref(nn), _ptr(boxes), _ptr(links),
                                          _ptr(order)))
        return boxes, links, order

    def vertex_normals(self, m: TriangleMesh) -> np.ndarray:
        out = np.zeros((m.vertex_count(), 3))
        v = m.view()
        self._check(self.fn("vertex_normals")(ctypes.byref(v), _ptr(out)))
        return out

    def wedge_tangents(self, m: TriangleMesh) -> np.ndarray:
        out = np.zeros((m.face_count(), 3, 3, 3))
        v = m.view()
        self._check(self.fn("wedge_tangents")(ctypes.byref(v), _ptr(out)))
        return out

    def baked_mean_error(self, lo: TriangleMesh, rgb: np.ndarray, res: int, hi: TriangleMesh,
                         samples: int = 10000, seed: int = 7):
        rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        mean, used, exc = ctypes.c_double(0), ctypes.c_int(0), ctypes.c_int(0)
        lv, hv = lo.view(), hi.view()
        self._check(self.fn("baked_mean_error")(ctypes.byref(lv), _ptr(rgb), ctypes.c_int(res),
                                                ctypes.c_int(res), ctypes.byref(hv), ctypes.c_int(samples),
                                                ctypes.c_uint64(seed), ctypes.byref(mean),
                                                ctypes.byref(used), ctypes.byref(exc)))
        return mean.value, used.value, exc.value

    def fixture(self, kind: int, a: int = 0, b: int = 0, c: int = 0, r: float = 0.5) -> TriangleMesh:
        nv, nf = ctypes.c_int(0), ctypes.c_int(0)
        self._check(self.fn("fixture_make")(ctypes.c_int(kind), ctypes.c_int(a), ctypes.c_int(b),
                                            ctypes.c_uint64(c), ctypes.c_double(r), ctypes.byref(nv),
                                            ctypes.byref(nf)))
        pos = np.zeros((nv.value, 3))
        faces = np.zeros((nf.value, 3), np.int32)
        self.fn("fixture_get")(_ptr(pos), _ptr(faces))
        return TriangleMesh(pos, faces)

    def random_points(self, n, lo, hi, seed):
        out = np.zeros((n, 3))
        box = np.array(list(lo) + list(hi), dtype=np.float64)
        self.fn("random_points")(ctypes.c_int(n), _ptr(box), ctypes.c_uint64(seed), _ptr(out))
        return out

    def random_units(self, n, seed):
        out = np.zeros((n, 3))
        self.fn("random_units")(ctypes.c_int(n), ctypes.c_uint64(seed), _ptr(out))
        return out


_port: Optional[Port] = None
_ref: Optional[Ref] = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port(PORT_LIB)
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref(REF_LIB)
    return _ref
