"""Deterministic synthetic meshes: the reference's test fixtures and the
benchmark family of SURVEY.md Appendix B.

Restated from ``proj/tests/support/fixtures.cpp`` (icosphere :17-54, uvSphere
:56-85, box :112-156, planeGrid :158-171, BlobField/starBlob :208-254,
randomPointsInBox/randomUnitVectors :336-358) and ``core/rng.h:10-29``
(CounterRng), plus the geodesic benchmark pairs G(n_dense) -> G(n_low) with a
20-chart UV atlas. These generate INPUTS only; both the CUDA path and the CPU
oracle consume the same arrays, so ulp-level differences from the reference's
own fixture code (numpy vs glibc sin/cos) cannot affect parity.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .mesh import TriangleMesh

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


# ---------------------------------------------------------------- CounterRng
def _mix(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser (rng.h:16-21), vectorised over uint64."""
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


class CounterRng:
    """Stateless counter RNG (rng.h:10-29): draw i = f(seed, i)."""

    def __init__(self, seed: int = 0):
        self.seed = np.uint64(seed)
        self._mseed = _mix(np.array([self.seed], dtype=np.uint64))[0]

    def bits(self, i) -> np.ndarray:
        i = np.asarray(i, dtype=np.uint64)
        with np.errstate(over="ignore"):
            return _mix(np.uint64(self._mseed) ^ _mix(i + np.uint64(0x632BE59BD9B4E019)))

    def uniform(self, i) -> np.ndarray:
        return (self.bits(i) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def below(self, i, n: int) -> np.ndarray:
        return self.bits(i) % np.uint64(n)


# ---------------------------------------------------------- reference fixtures
_T = (1.0 + math.sqrt(5.0)) / 2.0
ICO_POSITIONS = np.array(
    [[-1, _T, 0], [1, _T, 0], [-1, -_T, 0], [1, -_T, 0], [0, -1, _T], [0, 1, _T],
     [0, -1, -_T], [0, 1, -_T], [_T, 0, -1], [_T, 0, 1], [-_T, 0, -1], [-_T, 0, 1]],
    dtype=np.float64)
ICO_FACES = np.array(
    [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4],
     [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8],
     [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int32)


def _norm_rows(p: np.ndarray) -> np.ndarray:
    """Row norms with the pinned (x*x + y*y) + z*z order."""
    return np.sqrt((p[:, 0] * p[:, 0] + p[:, 1] * p[:, 1]) + p[:, 2] * p[:, 2])


def icosphere(subdivisions: int, radius: float = 0.5, center=(0.0, 0.0, 0.0)) -> TriangleMesh:
    """fixtures.cpp:17-54 (recursive midpoint subdivision, 20*4^k faces)."""
    pos = [tuple(p) for p in ICO_POSITIONS]
    faces = [tuple(f) for f in ICO_FACES]
    for _ in range(subdivisions):
        mids: dict = {}

        def midpoint(a, b):
            key = (a, b) if a < b else (b, a)
            idx = mids.get(key)
            if idx is None:
                idx = len(pos)
                mids[key] = idx
                pa, pb = pos[a], pos[b]
                pos.append(((pa[0] + pb[0]) * 0.5, (pa[1] + pb[1]) * 0.5, (pa[2] + pb[2]) * 0.5))
            return idx

        nxt = []
        for f in faces:
            ab = midpoint(f[0], f[1])
            bc = midpoint(f[1], f[2])
            ca = midpoint(f[2], f[0])
            nxt += [(f[0], ab, ca), (f[1], bc, ab), (f[2], ca, bc), (ab, bc, ca)]
        faces = nxt
    p = np.array(pos, dtype=np.float64)
    n = _norm_rows(p)
    p = np.asarray(center, dtype=np.float64) + (p / n[:, None]) * radius
    return TriangleMesh(p, np.array(faces, dtype=np.int32))


def uv_sphere(stacks: int, slices: int, radius: float = 0.5, center=(0.0, 0.0, 0.0)) -> TriangleMesh:
    """fixtures.cpp:56-85 (lat/long sphere, 2*slices*(stacks-1) faces)."""
    c = np.asarray(center, dtype=np.float64)
    pos = [c + np.array([0.0, 0.0, radius])]
    for s in range(1, stacks):
        theta = math.pi * s / stacks
        for l in range(slices):
            phi = 2.0 * math.pi * l / slices
            pos.append(c + radius * np.array([math.sin(theta) * math.cos(phi),
                                              math.sin(theta) * math.sin(phi), math.cos(theta)]))
    bottom = len(pos)
    pos.append(c + np.array([0.0, 0.0, -radius]))

    def ring(s, l):
        return 1 + (s - 1) * slices + (l % slices)

    faces = [(0, ring(1, l), ring(1, l + 1)) for l in range(slices)]
    for s in range(1, stacks - 1):
        for l in range(slices):
            a, b, cc, d = ring(s, l), ring(s, l + 1), ring(s + 1, l), ring(s + 1, l + 1)
            faces += [(a, cc, d), (a, d, b)]
    faces += [(bottom, ring(stacks - 1, l + 1), ring(stacks - 1, l)) for l in range(slices)]
    return TriangleMesh(np.array(pos), np.array(faces, dtype=np.int32))


def plane_grid(nx: int, ny: int, width: float = 1.0, height: float = 1.0) -> TriangleMesh:
    """fixtures.cpp:158-171."""
    pos = [(width * i / nx, height * j / ny, 0.0) for j in range(ny + 1) for i in range(nx + 1)]
    idx = lambda i, j: j * (nx + 1) + i  # noqa: E731
    faces = []
    for j in range(ny):
        for i in range(nx):
            faces += [(idx(i, j), idx(i + 1, j), idx(i + 1, j + 1)), (idx(i, j), idx(i + 1, j + 1), idx(i, j + 1))]
    return TriangleMesh(np.array(pos), np.array(faces, dtype=np.int32))


def box(half_extents=(0.5, 0.5, 0.5), n: int = 1) -> TriangleMesh:
    """fixtures.cpp:112-156 (n x n grid per side, deduplicated corners)."""
    h = np.asarray(half_extents, dtype=np.float64)
    sides = [
        ((h[0], -h[1], -h[2]), (0, 2 * h[1], 0), (0, 0, 2 * h[2])),
        ((-h[0], -h[1], -h[2]), (0, 0, 2 * h[2]), (0, 2 * h[1], 0)),
        ((-h[0], h[1], -h[2]), (0, 0, 2 * h[2]), (2 * h[0], 0, 0)),
        ((-h[0], -h[1], -h[2]), (2 * h[0], 0, 0), (0, 0, 2 * h[2])),
        ((-h[0], -h[1], h[2]), (2 * h[0], 0, 0), (0, 2 * h[1], 0)),
        ((-h[0], -h[1], -h[2]), (0, 2 * h[1], 0), (2 * h[0], 0, 0)),
    ]
    pos, faces, dedup = [], [], {}

    def vertex(p):
        key = tuple(int(round(p[k] / h[k] * n * 2)) for k in range(3))
        if key not in dedup:
            dedup[key] = len(pos)
            pos.append(p)
        return dedup[key]

    for o, du, dv in sides:
        o, du, dv = np.array(o), np.array(du), np.array(dv)
        for i in range(n):
            for j in range(n):
                p00 = o + du * (i / n) + dv * (j / n)
                p10 = o + du * ((i + 1) / n) + dv * (j / n)
                p01 = o + du * (i / n) + dv * ((j + 1) / n)
                p11 = o + du * ((i + 1) / n) + dv * ((j + 1) / n)
                a, b, c, d = vertex(p00), vertex(p10), vertex(p11), vertex(p01)
                faces += [(a, b, c), (a, c, d)]
    return TriangleMesh(np.array(pos), np.array(faces, dtype=np.int32))


class WaveField:
    """Sum of plane waves over directions: f(d) = sum_k amp_k sin(w_k d.a_k + phi_k).

    ``WaveField.blob(seed)`` is the reference BlobField (fixtures.cpp:208-236:
    5 waves, w in [2, 6], sum(amp) = 0.2, including its counter layout);
    ``WaveField.detail(seed)`` is the Appendix-B high-frequency detail field
    (24 waves, w in [40, 120], sum(amp) = 0.01).
    """

    def __init__(self, axis, freq, phase, amp):
        self.axis, self.freq, self.phase, self.amp = axis, freq, phase, amp

    @classmethod
    def blob(cls, seed: int) -> "WaveField":
        rng = CounterRng(seed)
        k = np.arange(5, dtype=np.uint64)
        z = 2.0 * rng.uniform(4 * k) - 1.0
        phi = 2.0 * math.pi * rng.uniform(4 * k + 1)
        s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
        axis = np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)
        freq = 2.0 + 4.0 * rng.uniform(4 * k + 2)
        phase = 2.0 * math.pi * rng.uniform(4 * k + 3)
        amp = 0.5 + rng.uniform(4 * k + 7)
        total = 0.0
        for a in amp:
            total += a
        return cls(axis, freq, phase, amp * (0.2 / total))

    @classmethod
    def detail(cls, seed: int, waves: int = 24, total_amp: float = 0.01) -> "WaveField":
        rng = CounterRng(seed)
        k = np.arange(waves, dtype=np.uint64)
        z = 2.0 * rng.uniform(5 * k) - 1.0
        phi = 2.0 * math.pi * rng.uniform(5 * k + 1)
        s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
        axis = np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)
        freq = 40.0 + 80.0 * rng.uniform(5 * k + 2)
        phase = 2.0 * math.pi * rng.uniform(5 * k + 3)
        amp = 0.5 + rng.uniform(5 * k + 4)
        return cls(axis, freq, phase, amp * (total_amp / amp.sum()))

    def eval(self, dirs: np.ndarray) -> np.ndarray:
        d = np.atleast_2d(dirs)
        f = np.zeros(d.shape[0])
        for k in range(len(self.amp)):
            a = self.axis[k]
            dot = (d[:, 0] * a[0] + d[:, 1] * a[1]) + d[:, 2] * a[2]
            f = f + self.amp[k] * np.sin(self.freq[k] * dot + self.phase[k])
        return f


def star_blob(seed: int, stacks: int, slices: int, base_radius: float = 0.5,
              center=(0.0, 0.0, 0.0)) -> TriangleMesh:
    """fixtures.cpp:245-254."""
    m = uv_sphere(stacks, slices, 1.0)
    d = m.positions / _norm_rows(m.positions)[:, None]
    field = WaveField.blob(seed)
    m.positions = np.ascontiguousarray(np.asarray(center) + d * (base_radius * (1.0 + field.eval(d)))[:, None])
    return m


def random_points_in_box(n: int, lo, hi, seed: int) -> np.ndarray:
    """fixtures.cpp:336-346."""
    rng = CounterRng(seed)
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    ext = hi - lo
    i = np.arange(n, dtype=np.uint64)
    u = np.stack([rng.uniform(3 * i) * ext[0], rng.uniform(3 * i + 1) * ext[1],
                  rng.uniform(3 * i + 2) * ext[2]], axis=1)
    return lo + u


def random_unit_vectors(n: int, seed: int) -> np.ndarray:
    """fixtures.cpp:348-358."""
    rng = CounterRng(seed)
    i = np.arange(n, dtype=np.uint64)
    z = 2.0 * rng.uniform(2 * i) - 1.0
    phi = 2.0 * math.pi * rng.uniform(2 * i + 1)
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)


def identity_quad() -> TriangleMesh:
    """test_bake.cpp:39-46: z=0 quad whose UVs equal its xy."""
    return TriangleMesh([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], [[0, 1, 2], [0, 2, 3]],
                        uvs=[[0, 0], [1, 0], [1, 1], [0, 1]], face_uvs=[[0, 1, 2], [0, 2, 3]])


def assign_cell_uvs(mesh: TriangleMesh, columns: int) -> TriangleMesh:
    """test_metrics.cpp:55-71: one UV island per face on a grid."""
    nf = mesh.face_count()
    rows = (nf + columns - 1) // columns
    cw, ch = 1.0 / columns, 1.0 / rows
    f = np.arange(nf)
    u0 = (f % columns) * cw + 0.1 * cw
    v0 = (f // columns) * ch + 0.1 * ch
    uvs = np.stack([np.stack([u0, v0], 1), np.stack([u0 + 0.8 * cw, v0], 1),
                    np.stack([u0, v0 + 0.8 * ch], 1)], axis=1).reshape(-1, 2)
    mesh.uvs = np.ascontiguousarray(uvs)
    mesh.face_uvs = np.ascontiguousarray(np.arange(3 * nf, dtype=np.int32).reshape(-1, 3))
    return mesh


# ------------------------------------------------- Appendix B benchmark family
def _geodesic_topology(n: int):
    """Topology of G(n): the icosahedron with each face split into n^2
    triangles on the barycentric grid (i, j) -> weights (n-i-j, i, j)/n over
    the face corners (A, B, C); shared edge/corner vertices deduplicated.
    Returns (vertex_weights, faces, face_grid) where vertex_weights is a
    list of (corner_a, corner_b, corner_c, wa, wb, wc) rows describing each
    vertex as an exact integer combination of icosahedron corners, and
    face_grid[f] = (ico_face, grid indices of its 3 corners)."""
    # unique edges in first-appearance order
    edge_base: dict = {}
    nxt = 12
    for f in ICO_FACES:
        for k in range(3):
            a, b = int(f[k]), int(f[(k + 1) % 3])
            key = (min(a, b), max(a, b))
            if key not in edge_base:
                edge_base[key] = nxt
                nxt += n - 1
    n_edge_end = nxt
    interior_per_face = (n - 1) * (n - 2) // 2
    nv = n_edge_end + 20 * interior_per_face
    assert nv == 10 * n * n + 2

    gi, gj, tri_grid = _geodesic_topology_grid(n)
    gid_count = gi.size

    vert_corner = np.zeros((nv, 3), dtype=np.int64)   # three ico corners
    vert_w = np.zeros((nv, 3), dtype=np.int64)        # integer weights summing to n
    vert_corner[:12] = np.arange(12)[:, None]
    vert_w[:12, 0] = n
    for (a, b), base in edge_base.items():
        s = np.arange(1, n)
        idx = base + s - 1
        vert_corner[idx] = [a, b, b]
        vert_w[idx, 0] = n - s
        vert_w[idx, 1] = s
    gmap = np.zeros((20, gid_count), dtype=np.int64)
    for f in range(20):
        A, B, C = (int(x) for x in ICO_FACES[f])
        ids = np.empty(gi.size, dtype=np.int64)
        wa = n - gi - gj
        # corners
        ids[(gi == 0) & (gj == 0)] = A
        ids[(gi == n)] = B
        ids[(gj == n)] = C

        def edge_ids(u, v, s):
            if u < v:
                return edge_base[(u, v)] + s - 1
            return edge_base[(v, u)] + (n - s) - 1

        e_ab = (gj == 0) & (gi > 0) & (gi < n)
        ids[e_ab] = edge_ids(A, B, gi[e_ab])
        e_ac = (gi == 0) & (gj > 0) & (gj < n)
        ids[e_ac] = edge_ids(A, C, gj[e_ac])
        e_bc = (gi + gj == n) & (gi > 0) & (gj > 0)
        ids[e_bc] = edge_ids(B, C, gj[e_bc])
        inner = (gi > 0) & (gj > 0) & (gi + gj < n)
        base = n_edge_end + f * interior_per_face
        ids[inner] = base + np.arange(int(inner.sum()))
        vert_corner[ids[inner]] = [A, B, C]
        vert_w[ids[inner]] = np.stack([wa[inner], gi[inner], gj[inner]], 1)
        gmap[f] = ids
    faces = np.concatenate([gmap[f][tri_grid] for f in range(20)], 0).astype(np.int32)
    return vert_corner, vert_w, faces, (gi, gj, tri_grid)


def geodesic_directions(n: int):
    """Unit directions and faces of G(n) (F = 20 n^2, V = 10 n^2 + 2)."""
    vc, vw, faces, grid = _geodesic_topology(n)
    p = (ICO_POSITIONS[vc[:, 0]] * vw[:, 0:1] + ICO_POSITIONS[vc[:, 1]] * vw[:, 1:2]
         + ICO_POSITIONS[vc[:, 2]] * vw[:, 2:3]) / float(n)
    d = p / _norm_rows(p)[:, None]
    return d, faces, grid


def chart_atlas(n: int, res: int, margin_texels: float = 3.0):
    """The 20-chart atlas of Appendix B: one equilateral chart per icosahedron
    face, 4 rows x 5 alternating up/down triangles, each shrunk so that
    neighbouring charts are >= 2*margin_texels apart at ``res``. Returns
    (uvs, face_uvs) for G(n)'s face order; interior wedges of a chart share
    one UV index per grid point (as unwrapMesh does, unwrap.cpp:54-73)."""
    gi, gj, tri_grid = _geodesic_topology_grid(n)
    pad = 0.01
    L = (1.0 - 2 * pad) / (4 * math.sqrt(3.0) / 2.0)
    H = L * math.sqrt(3.0) / 2.0
    r_in = L / (2.0 * math.sqrt(3.0))
    margin_texels = min(margin_texels, 0.25 * r_in * res)  # small atlases: keep charts >= 3/4 size
    delta = margin_texels / res
    shrink = (r_in - delta) / r_in
    assert shrink > 0.5, "atlas resolution too small for the chart margin"
    npts = gi.size
    uvs = np.zeros((20 * npts, 2))
    face_uvs = np.zeros((20 * tri_grid.shape[0], 3), dtype=np.int32)
    for f in range(20):
        row, slot = divmod(f, 5)
        x0, y0 = pad, pad + row * H
        m = slot // 2
        if slot % 2 == 0:
            A = np.array([x0 + m * L, y0 + H])
            B = np.array([x0 + (m + 1) * L, y0 + H])
            C = np.array([x0 + m * L + L / 2, y0])
        else:
            A = np.array([x0 + m * L + L / 2, y0])
            B = np.array([x0 + (m + 1) * L, y0 + H])
            C = np.array([x0 + (m + 1) * L + L / 2, y0])
        cen = (A + B + C) / 3.0
        A, B, C = (cen + (P - cen) * shrink for P in (A, B, C))
        wa = (n - gi - gj)[:, None] / n
        uvs[f * npts:(f + 1) * npts] = A * wa + B * (gi[:, None] / n) + C * (gj[:, None] / n)
        face_uvs[f * tri_grid.shape[0]:(f + 1) * tri_grid.shape[0]] = tri_grid + f * npts
    return uvs, face_uvs


def _geodesic_topology_grid(n: int):
    ii, jj = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    keep = ii + jj <= n
    gi, gj = ii[keep], jj[keep]
    gid = -np.ones((n + 1, n + 1), dtype=np.int64)
    gid[gi, gj] = np.arange(gi.size)
    ui, uj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    m = ui + uj <= n - 1
    ui, uj = ui[m], uj[m]
    up = np.stack([gid[ui, uj], gid[ui + 1, uj], gid[ui, uj + 1]], 1)
    m2 = ui + uj <= n - 2
    di, dj = ui[m2], uj[m2]
    down = np.stack([gid[di + 1, dj], gid[di + 1, dj + 1], gid[di, dj + 1]], 1)
    tri_grid = np.concatenate([up, down], 0)
    order = np.lexsort((np.concatenate([np.zeros(len(up)), np.ones(len(down))]),
                        np.concatenate([uj, dj]), np.concatenate([ui, di])))
    return gi, gj, tri_grid[order]


@dataclass
class BakePair:
    name: str
    dense: TriangleMesh
    lowpoly: TriangleMesh
    res: int
    max_distance_fraction: float
    radius: int = 4

    _diag: float = -1.0

    @property
    def bbox_diagonal(self) -> float:
        """bounds(dense).diagonal() (test_bake.cpp:206), computed once."""
        if self._diag < 0:
            self._diag = self.dense.bbox_diagonal()
        return self._diag


# BASELINE.json configs (SURVEY §8 sizes table / BASELINE.md §2 inputs)
CONFIGS = {
    "A": dict(n_dense=100, n_low=16, res=512, frac=0.01, seed=7, low_scale=1.0),
    "B": dict(n_dense=224, n_low=32, res=2048, frac=0.01, seed=7, low_scale=1.0),
    "C": dict(n_dense=224, n_low=32, res=4096, frac=0.01, seed=7, low_scale=1.0),
    "D": dict(n_dense=158, n_low=22, res=1024, frac=0.01, seed=100, low_scale=1.0),
    "E": dict(n_dense=447, n_low=50, res=4096, frac=0.05, seed=7, low_scale=1.04),
}


def bake_pair(n_dense: int, n_low: int, res: int, frac: float = 0.01, seed: int = 7,
              low_scale: float = 1.0, name: str = "custom", detail: bool = True) -> BakePair:
    """Dense G(n_dense) displaced by f_lo + f_hi, lowpoly G(n_low) on the f_lo
    surface (times low_scale, the "cage offset" of config E) with the 20-chart
    atlas at ``res``."""
    lo_field = WaveField.blob(seed)
    d_dirs, d_faces, _ = geodesic_directions(n_dense)
    r = lo_field.eval(d_dirs)
    if detail:
        r = r + WaveField.detail(seed + 1000).eval(d_dirs)
    dense = TriangleMesh(d_dirs * (0.5 * (1.0 + r))[:, None], d_faces)
    l_dirs, l_faces, _ = geodesic_directions(n_low)
    lr = 0.5 * (1.0 + lo_field.eval(l_dirs)) * low_scale
    uvs, face_uvs = chart_atlas(n_low, res)
    lowpoly = TriangleMesh(l_dirs * lr[:, None], l_faces, uvs=uvs, face_uvs=face_uvs)
    return BakePair(name, dense, lowpoly, res, frac)


def config_pair(name: str, seed: int | None = None) -> BakePair:
    c = dict(CONFIGS[name])
    if seed is not None:
        c["seed"] = seed
    return bake_pair(c["n_dense"], c["n_low"], c["res"], c["frac"], c["seed"], c["low_scale"], name=name)
