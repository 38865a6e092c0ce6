"""GPU: the LBVH queries (Bvh::closestPointWithin / raycastFirst and the
brute-force oracles) through the C ABI, restating proj/tests/test_spatial.cpp
and checking against reference goldens: face ids, distances, points, t/u/v
bit-exact."""
import os

import numpy as np
import pytest

from paper_2605_26137_b200 import fixtures as fx
from paper_2605_26137_b200 import meshforge as mf
from paper_2605_26137_b200.mesh import TriangleMesh

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def brute_closest(ctx, mesh, q):
    import ctypes
    q = np.ascontiguousarray(q, np.float64).reshape(-1, 3)
    n = q.shape[0]
    f, d, p, b = np.zeros(n, np.int32), np.zeros(n), np.zeros((n, 3)), np.zeros((n, 3))
    v = mesh.view()
    from paper_2605_26137_b200.capi import check
    P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    check(ctx.lib.mf_closest_point_brute(ctx.h, ctypes.byref(v), P(q), n, P(f), P(d), P(p), P(b)))
    return f, d, p, b


def brute_ray(ctx, mesh, o, dr, tmin=0.0, tmax=float("inf")):
    import ctypes
    o = np.ascontiguousarray(o, np.float64).reshape(-1, 3)
    dr = np.ascontiguousarray(dr, np.float64).reshape(-1, 3)
    n = o.shape[0]
    f, t, u, v_ = np.zeros(n, np.int32), np.zeros(n), np.zeros(n), np.zeros(n)
    v = mesh.view()
    from paper_2605_26137_b200.capi import check
    P = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    check(ctx.lib.mf_raycast_first_brute(ctx.h, ctypes.byref(v), P(o), P(dr), n, tmin, tmax, P(f), P(t), P(u),
                                         P(v_)))
    return f, t, u, v_


def test_golden_closest_points_and_rays(gpu_ctx):
    d = np.load(os.path.join(GOLDEN, "spatial.npz"))
    ico = TriangleMesh(d["ico_pos"], d["ico_faces"])
    bvh = mf.Bvh(ico)
    f, ds, pt, bary = bvh.closest_points(d["q"])
    assert np.array_equal(f, d["cp_face"]) and np.array_equal(ds, d["cp_dist"])
    assert np.array_equal(pt, d["cp_point"]) and np.array_equal(bary, d["cp_bary"])
    f, ds, _, _ = bvh.closest_points(d["q"], 0.2)
    assert np.array_equal(f, d["cpw_face"]) and np.array_equal(ds, d["cpw_dist"])
    uvs = TriangleMesh(d["uvs_pos"], d["uvs_faces"])
    f, t, u, v = mf.Bvh(uvs).raycasts(d["ray_o"], d["ray_d"])
    assert np.array_equal(f, d["ray_face"])
    hit = f >= 0
    assert np.array_equal(t[hit], d["ray_t"][hit])
    assert np.array_equal(u[hit], d["ray_u"][hit]) and np.array_equal(v[hit], d["ray_v"][hit])


def test_bvh_equals_brute_force_rays_10k_sphere(gpu_ctx, port):
    """test_spatial.cpp:139-161 (bit-exact face, t, u, v), plus the oracle."""
    sphere = fx.uv_sphere(72, 72, 0.5)
    assert sphere.face_count() > 10000
    o = fx.random_points_in_box(1000, (-1.5,) * 3, (1.5,) * 3, 21)
    dirs = fx.random_unit_vectors(1000, 22)
    tgt = fx.random_points_in_box(1000, (-0.4,) * 3, (0.4,) * 3, 23)
    aim = (tgt - o) / np.linalg.norm(tgt - o, axis=1, keepdims=True)
    dirs[::2] = aim[::2]
    a = mf.Bvh(sphere).raycasts(o, dirs)
    b = brute_ray(gpu_ctx, sphere, o, dirs)
    c = port.raycast_first(sphere, o, dirs, brute=True)
    for x, y, z in zip(a, b, c):
        assert np.array_equal(x, y) and np.array_equal(x, z)
    assert (a[0] >= 0).sum() > 100


def test_closest_point_equals_brute_force(gpu_ctx, port):
    """test_spatial.cpp:184-195 on starBlob(4, 48, 48), 1000 queries."""
    blob = fx.star_blob(4, 48, 48)
    q = fx.random_points_in_box(1000, (-1,) * 3, (1,) * 3, 31)
    a = mf.Bvh(blob).closest_points(q)
    b = brute_closest(gpu_ctx, blob, q)
    c = port.closest_within(blob, q, brute=True)
    for x, y, z in zip(a, b, c):
        assert np.array_equal(x, y) and np.array_equal(x, z)


def test_bounded_matches_global_inside_radius(gpu_ctx):
    """test_spatial.cpp:197-212."""
    s = fx.icosphere(3)
    q = fx.random_points_in_box(200, (-1,) * 3, (1,) * 3, 41)
    bvh = mf.Bvh(s)
    fa, da, _, _ = bvh.closest_points(q)
    fb, db, _, _ = bvh.closest_points(q, 0.2)
    inside, outside = np.sqrt(da) < 0.2, np.sqrt(da) > 0.2
    assert np.array_equal(fb[inside], fa[inside]) and np.array_equal(db[inside], da[inside])
    assert (fb[outside] == -1).all() and np.isinf(db[outside]).all()


def test_small_known_answers(gpu_ctx):
    """test_spatial.cpp:74-137,163-182,214-226."""
    tri = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    h = mf.Bvh(tri).raycast_first([1 / 3, 1 / 3, 2.0], [0, 0, -1])
    assert h.valid() and h.face == 0 and abs(h.t - 2.0) < 1e-12
    cube = fx.box((0.5, 0.5, 0.5))
    h = mf.Bvh(cube).raycast_first([2, 0.1, 0.1], [-1, 0, 0])
    assert h.valid() and abs(h.t - 1.5) < 1e-12
    assert np.allclose(cube.positions[cube.faces[h.face]][:, 0], 0.5)
    assert not mf.Bvh(fx.plane_grid(2, 2)).raycast_first([-1, -1, 0.5], [1, 0, 0]).valid()
    quad = TriangleMesh([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], [[0, 1, 2], [0, 2, 3]])
    assert mf.Bvh(quad).raycast_first([0.25, 0.25, 1.0], [0, 0, -1]).face == 0  # lower face on the tie
    s = fx.icosphere(1)
    sp = mf.Bvh(s).closest_point(s.positions[7])
    assert sp.valid() and sp.distance() < 1e-12 and abs(sp.barycentric.max() - 1.0) < 1e-12
    assert abs(mf.Bvh(fx.box((0.5, 0.5, 0.5), 2)).closest_point([0, 0, 0]).distance() - 0.5) < 1e-12
    s2 = fx.icosphere(2)
    rng = fx.CounterRng(6)
    bvh = mf.Bvh(s2)
    for i in range(100):
        f = int(rng.below(3 * i, s2.face_count()))
        u = float(rng.uniform(3 * i + 1))
        v = float(rng.uniform(3 * i + 2)) * (1 - u)
        t = s2.positions[s2.faces[f]]
        p = (1 - u - v) * t[0] + u * t[1] + v * t[2]
        assert bvh.closest_point(p).distance() < 1e-9


def test_bvh_export_structurally_sound(gpu_ctx):
    """test_spatial.cpp:228-263: every face in exactly one leaf, leaf boxes
    contain their triangles, deterministic build."""
    m = fx.star_blob(9, 40, 40)
    a, b = mf.Bvh(m).export(), mf.Bvh(m).export()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    boxes, links, order = a
    leaf = links[:, 3] > 0
    seen = np.concatenate([order[f:f + c] for f, c in links[leaf][:, 2:4]])
    assert np.array_equal(np.sort(seen), np.arange(m.face_count()))
    for (f, c), box in zip(links[leaf][:, 2:4], boxes[leaf]):
        pts = m.positions[m.faces[order[f:f + c]]].reshape(-1, 3)
        assert (pts >= box[:3] - 1e-12).all() and (pts <= box[3:] + 1e-12).all()


def test_bvh_rejects_bad_input(gpu_ctx):
    """test_spatial.cpp:265-274."""
    with pytest.raises(mf.MeshforgeError):
        mf.Bvh(TriangleMesh([[0, 0, 0]], np.zeros((0, 3))))
    with pytest.raises(mf.MeshforgeError):
        mf.Bvh(TriangleMesh([[0, 0, 0], [1, 0, 0], [0, np.nan, 0]], [[0, 1, 2]]))


@pytest.mark.parametrize("case", ["ico4", "plane", "torus", "domain"])
def test_surface_band_matches_reference_golden(gpu_ctx, case):
    """markSurfaceBand's voxel sweep on the device (mf_surface_band): labels,
    f32 distances and the grid parameters bit-exact vs the reference build."""
    d = np.load(os.path.join(GOLDEN, "band.npz"))
    mesh = TriangleMesh(d[f"{case}_pos"], d[f"{case}_faces"])
    res, band, dil = d[f"{case}_params"]
    dom = d[f"{case}_domain"]
    labels, dist, grid = mf.Bvh(mesh).surface_band(int(res), float(band), int(dil),
                                                   None if np.isnan(dom).any() else dom)
    assert np.array_equal(labels, d[f"{case}_labels"])
    assert np.array_equal(dist.view(np.uint32), d[f"{case}_dist"].view(np.uint32))
    assert np.array_equal(np.r_[grid["origin"], grid["voxel_size"], grid["truncation"]], d[f"{case}_grid"])


def test_surface_band_dense_blob_matches_port(gpu_ctx, port):
    """A config-A-sized dense mesh (200k faces) on a 96^3 grid vs the oracle."""
    pair = fx.config_pair("A")
    m = pair.dense
    labels, dist, grid = mf.Bvh(m).surface_band(96, 1.0, 2)
    pl, pd, pg = port.surface_band(m, 96, 1.0, 2)
    assert np.array_equal(labels, pl)
    assert np.array_equal(dist.view(np.uint32), pd.view(np.uint32))
    assert labels.sum() > 1000


def test_surface_band_errors(gpu_ctx):
    from paper_2605_26137_b200.capi import MeshforgeError
    d = np.load(os.path.join(GOLDEN, "band.npz"))
    bvh = mf.Bvh(TriangleMesh(d["domain_pos"], d["domain_faces"]))
    for args, code in [((7, 1.0, 2, None), 12), ((32, 1.0, -1, None), 12), ((12, 1.0, 2, None), 12),
                       ((32, 1.0, 2, (0, 0, 0, 1, 1, 1)), 3)]:
        with pytest.raises(MeshforgeError) as e:
            bvh.surface_band(*args)
        assert e.value.status == code


def _deep_tree_mesh():
    """Karras worst case: 20k copies of one triangle (identical Morton keys:
    the hierarchy splits on index bits only) plus triangles whose centroids
    halve their distance to the origin along every axis (Morton keys sharing
    ever longer prefixes), so root-to-leaf paths run through both key parts."""
    tris = []
    base = np.array([[0.0, 0.0, 0.0], [1e-3, 0.0, 0.0], [0.0, 1e-3, 0.0]])
    tris += [base] * 20000
    for k in range(40):
        s = 2.0 ** -k
        tris.append(base * s + s)
        tris.append(base * s - s)
    pos = np.concatenate(tris, 0)
    faces = np.arange(pos.shape[0], dtype=np.int32).reshape(-1, 3)
    return TriangleMesh(pos, faces)


def test_deep_degenerate_tree_matches_brute_force(gpu_ctx):
    m = _deep_tree_mesh()
    bvh = mf.Bvh(m)
    _, _, depth = bvh.info()
    assert 16 <= depth <= 58
    rng = np.random.default_rng(5)
    q = np.concatenate([rng.uniform(-1, 1, (3000, 3)), rng.uniform(-1e-3, 2e-3, (3000, 3))])
    f, ds, pt, bary = bvh.closest_points(q)
    bf, bd, bp, bb = brute_closest(gpu_ctx, m, q)
    assert np.array_equal(f, bf) and np.array_equal(ds, bd)
    assert np.array_equal(pt, bp) and np.array_equal(bary, bb)
    d = rng.normal(size=(3000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rf, rt, _, _ = bvh.raycasts(q[:3000], d)
    xf, xt, _, _ = brute_ray(gpu_ctx, m, q[:3000], d)
    assert np.array_equal(rf, xf) and np.array_equal(rt[rf >= 0], xt[rf >= 0])


def test_bvh_outlives_its_context_and_serves_threads(gpu_ctx):
    """A tree built on a context stays usable after that context is destroyed
    (it owns its arrays, scratch and stream), and concurrent const queries
    from several host threads give the serial answers (bvh.h:28)."""
    import concurrent.futures as cf

    from paper_2605_26137_b200 import capi
    m = fx.icosphere(5)
    ctx = capi.Context(0)
    bvh = mf.Bvh(m, ctx=ctx)
    ctx.close()
    rng = np.random.default_rng(9)
    qs = [rng.uniform(-0.7, 0.7, (20000 + 1000 * i, 3)) for i in range(8)]
    serial = [bvh.closest_points(q, 0.05) for q in qs]
    with cf.ThreadPoolExecutor(max_workers=8) as pool:
        par = list(pool.map(lambda q: bvh.closest_points(q, 0.05), qs))
    for a, b in zip(serial, par):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def _morton30(m: TriangleMesh) -> np.ndarray:
    """lbvh.cu k_morton restated in numpy (same f64 operations): 10 bits per
    axis of the face centroid over the vertex bounds."""
    p = m.positions
    lo, hi = p.min(0), p.max(0)
    ext = hi - lo
    inv = np.where(ext > 0.0, 1023.0 / np.where(ext > 0.0, ext, 1.0), 0.0)
    f = m.faces
    c = ((p[f[:, 0]] + p[f[:, 1]]) + p[f[:, 2]]) / 3.0
    q = np.clip((c - lo) * inv, 0.0, 1023.0).astype(np.uint32)

    def spread(v):
        v = v & 0x3FF
        v = (v | (v << 16)) & 0x030000FF
        v = (v | (v << 8)) & 0x0300F00F
        v = (v | (v << 4)) & 0x030C30C3
        v = (v | (v << 2)) & 0x09249249
        return v

    return (spread(q[:, 0]) << 2) | (spread(q[:, 1]) << 1) | spread(q[:, 2])


@pytest.mark.parametrize("kind", ["blob", "dense", "dups", "tiny"])
def test_lbvh_leaf_order_is_the_stable_morton_sort(gpu_ctx, kind):
    """The hand-written 3-pass radix sort (sort.cu) is a stable sort of the
    30-bit Morton keys: the tree's leaf order equals numpy's stable argsort,
    across several 8192-key tiles, a partial last tile, and many equal keys
    (duplicated triangles: deep equal-key runs resolved by face index)."""
    if kind == "blob":
        m = fx.star_blob(9, 40, 40)
    elif kind == "dense":
        m = fx.bake_pair(96, 4, 16, name="sort").dense  # ~184k faces, 23 tiles
    elif kind == "dups":
        base = fx.star_blob(5, 24, 24)
        k = 40  # 40 copies of every face: equal keys in runs of 40
        m = TriangleMesh(base.positions, np.tile(base.faces, (k, 1)))
    else:
        m = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], [[0, 1, 2], [1, 3, 2]])
    _, _, order = mf.Bvh(m).export()
    expect = np.argsort(_morton30(m), kind="stable")
    assert np.array_equal(order, expect)
    if kind == "dups":  # the traversal copes with the deep equal-key subtrees
        b = mf.Bvh(m)
        q = np.random.default_rng(1).uniform(-0.6, 0.6, (2000, 3))
        f, ds, _, _ = b.closest_points(q)
        ref_f, ref_ds, _, _ = mf.Bvh(TriangleMesh(m.positions, m.faces[: len(m.faces) // 40])).closest_points(q)
        assert np.array_equal(ds, ref_ds)
        assert np.array_equal(f, ref_f)  # ties go to the lowest face index: the first copy


def test_sample_sdf_matches_reference(gpu_ctx, ref):
    """sampleSdf (signfield/watertight.cpp:29-38) batched on the device
    (mf_sample_sdf): bit-exact vs the reference's own function over the same
    mesh, grid geometry and signed field (a synthetic field: the signed
    distance to a sphere, sampled at the voxel centres)."""
    m = fx.star_blob(7, 32, 32)
    res = 24
    origin = np.array([-0.8, -0.75, -0.7])
    h = 1.5 / res
    c = origin + h * (np.stack(np.meshgrid(np.arange(res), np.arange(res), np.arange(res), indexing="ij"), -1) + 0.5)
    field = (np.linalg.norm(c, axis=-1) - 0.45).astype(np.float32).transpose(2, 1, 0).reshape(-1)  # x fastest
    rng = np.random.default_rng(9)
    pts = np.vstack([rng.uniform(-1.0, 1.0, (3000, 3)), [[0.0, 0.0, 0.0], [5.0, 5.0, 5.0], [-3.0, 0.1, 0.2]]])
    got = mf.Bvh(m).sample_sdf(res, origin, h, field, pts)
    exp = ref.sample_sdf(m, res, origin, h, field, pts)
    assert np.array_equal(got, exp)
    assert (got < 0).any() and (got > 0).any()
