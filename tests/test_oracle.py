"""CPU: pin the oracle (the plain-C restatement, oracle/mf_oracle.c) against
the reference.

1. Golden vectors in tests/golden/*.npz were produced by the reference's own
   translation units (tests/golden/make_golden.py over oracle/_ref); the port
   must reproduce them bit-for-bit (RGB, hit faces, pre-quantisation ts,
   G-buffer, closest points, ray hits, tangent frames).
2. When oracle/_ref is built (this container), the port is also compared live
   against the reference on fresh inputs, and the reference's own
   tests/test_spatial.cpp binary is run.
"""
import os
import subprocess

import numpy as np
import pytest

from paper_2605_26137_b200 import fixtures as fx
from paper_2605_26137_b200.mesh import TriangleMesh

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def u32(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.parametrize("case", ["tiny", "small", "cage"])
def test_port_matches_reference_golden_bake(port, case):
    d = load(f"bake_{case}.npz")
    p = fx.bake_pair(int(d["n_dense"]), int(d["n_low"]), int(d["res"]), float(d["frac"]), int(d["seed"]),
                     float(d["low_scale"]), name=case)
    assert p.bbox_diagonal == float(d["diag"])
    g = port.raster_gbuffer(p.lowpoly, int(d["res"]))
    assert np.array_equal(g.valid, d["valid"])
    assert np.array_equal(g.reliable, d["reliable"])
    for k in ("position", "normal", "tangent", "bitangent"):
        assert np.array_equal(u32(getattr(g, k)), u32(d[k])), k
    out = port.bake(p.lowpoly, p.dense, int(d["res"]), p.bbox_diagonal, float(d["frac"]), 4, debug=True)
    assert np.array_equal(out["face"], d["face"])
    assert np.array_equal(out["ts"].view(np.uint64), d["ts"].view(np.uint64))
    assert np.array_equal(out["rgb_raw"], d["rgb_raw"])
    assert np.array_equal(out["rgb"], d["rgb"])


def test_port_matches_reference_golden_spatial(port):
    d = load("spatial.npz")
    ico = TriangleMesh(d["ico_pos"], d["ico_faces"])
    f, ds, pt, bary = port.closest_within(ico, d["q"])
    assert np.array_equal(f, d["cp_face"])
    assert np.array_equal(ds, d["cp_dist"])
    assert np.array_equal(pt, d["cp_point"])
    assert np.array_equal(bary, d["cp_bary"])
    f, ds, _, _ = port.closest_within(ico, d["q"], 0.2)
    assert np.array_equal(f, d["cpw_face"])
    assert np.array_equal(ds, d["cpw_dist"])
    uvs = TriangleMesh(d["uvs_pos"], d["uvs_faces"])
    f, t, u, v = port.raycast_first(uvs, d["ray_o"], d["ray_d"])
    assert np.array_equal(f, d["ray_face"])
    hit = f >= 0
    assert hit.sum() > 50
    assert np.array_equal(t[hit], d["ray_t"][hit])
    assert np.array_equal(u[hit], d["ray_u"][hit]) and np.array_equal(v[hit], d["ray_v"][hit])


def test_port_matches_reference_golden_tangents(port):
    d = load("tangents.npz")
    m = TriangleMesh(d["pos"], d["faces"], uvs=d["uvs"], face_uvs=d["face_uvs"])
    assert np.array_equal(port.wedge_tangents(m), d["frames"])
    vm = TriangleMesh(d["vn_mesh_pos"], d["vn_mesh_faces"])
    assert np.array_equal(port.vertex_normals(vm), d["vnormals"])


def test_port_matches_reference_golden_kats(port):
    d = load("kats.npz")
    m = TriangleMesh([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [1, 0, 200]], [[0, 1, 2], [0, 2, 3], [1, 4, 2]],
                     uvs=[[0.05, 0.05], [0.35, 0.05], [0.35, 0.35], [0.05, 0.35], [0.65, 0.05]],
                     face_uvs=[[0, 1, 2], [0, 2, 3], [1, 4, 2]])
    g = port.raster_gbuffer(m, 128)
    assert np.array_equal(g.valid, d["od_valid"]) and np.array_equal(g.reliable, d["od_reliable"])
    assert (g.valid & (1 - g.reliable)).sum() > 0  # the stretched face is unreliable
    assert np.array_equal(port.transfer_normals(g, m, m.bbox_diagonal()), d["od_rgb"])
    q, far = fx.identity_quad(), fx.identity_quad()
    far.positions[:, 2] += 0.08
    g = port.raster_gbuffer(q, 32)
    rgb = port.transfer_normals(g, far, float(np.sqrt(2.0)))
    assert np.array_equal(rgb, d["far_rgb"])
    assert (rgb[g.valid == 1] == [128, 128, 255]).all()
    fill = port.raster_gbuffer(q, 8).valid
    assert np.array_equal(fill, d["fill_valid"]) and fill.sum() == 64
    tri = TriangleMesh([[0, 0, 0], [2, 0, 0], [0, 2, 0]], [[0, 1, 2]], uvs=[[0, 0], [2, 0], [0, 2]],
                       face_uvs=[[0, 1, 2]])
    g = port.raster_gbuffer(tri, 32)
    assert np.array_equal(u32(g.position), u32(d["tri_position"]))
    assert np.array_equal(u32(g.normal), u32(d["tri_normal"]))
    out = port.dilate_seams(d["lone_in"], 11, 11, 3, 11, d["lone_valid"], 2)
    assert np.array_equal(out, d["lone_out"])


def test_port_error_codes(port):
    """test_bake.cpp:332-350 error codes (1 + ErrorCode)."""
    from oracle.bindings import OracleError
    bare = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    with pytest.raises(OracleError) as e:
        port.raster_gbuffer(bare, 64)
    assert e.value.code == 2  # InvalidGeometry
    with pytest.raises(OracleError) as e:
        port.raster_gbuffer(fx.identity_quad(), 0)
    assert e.value.code == 12  # InvalidConfig
    overlap = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [0, 1, 1]],
                           [[0, 1, 2], [3, 4, 5]],
                           uvs=[[0.1, 0.1], [0.9, 0.1], [0.1, 0.9], [0.2, 0.2], [0.8, 0.2], [0.2, 0.8]],
                           face_uvs=[[0, 1, 2], [3, 4, 5]])
    with pytest.raises(OracleError) as e:
        port.raster_gbuffer(overlap, 64)
    assert e.value.code == 8  # AtlasOverlap
    g = port.raster_gbuffer(fx.identity_quad(), 16)
    with pytest.raises(OracleError) as e:
        port.transfer_normals(g, fx.identity_quad(), 0.0)
    assert e.value.code == 12
    with pytest.raises(OracleError) as e:
        port.dilate_seams(np.zeros((64, 3), np.uint8), 8, 8, 3, 16, g.valid, 2)
    assert e.value.code == 9  # ShapeMismatch
    with pytest.raises(OracleError) as e:
        port.dilate_seams(np.zeros((256, 3), np.uint8), 16, 16, 3, 16, g.valid, -1)
    assert e.value.code == 12


# ---------------------------------------------------------------- live vs the reference
def test_port_matches_reference_live_bake(port, ref):
    p = fx.bake_pair(40, 6, 96, 0.02, 3, 1.01, name="live")
    a = port.bake(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 3, debug=True)
    b = ref.bake(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 3, debug=True)
    assert np.array_equal(a["face"], b["face"])
    assert np.array_equal(a["ts"].view(np.uint64), b["ts"].view(np.uint64))
    assert np.array_equal(a["rgb"], b["rgb"])


def test_port_matches_reference_live_spatial(port, ref):
    blob = ref.fixture(2, 48, 48, c=4, r=0.5)  # starBlob(4, 48, 48), test_spatial.cpp:184-195
    q = ref.random_points(500, (-1, -1, -1), (1, 1, 1), 31)
    for brute in (False, True):
        a = port.closest_within(blob, q, brute=brute)
        b = ref.closest_within(blob, q, brute=brute)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    cube = ref.fixture(3, 1, r=0.5)
    o = np.tile([0.01, -0.02, 0.03], (64, 1))
    d = ref.random_units(64, 3)
    a = port.raycast_first(cube, o, d)
    b = ref.raycast_first(cube, o, d, brute=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_fixture_restatements_match_reference(ref):
    for k in (0, 1, 3):
        a, b = fx.icosphere(k), ref.fixture(0, k, r=0.5)
        assert np.array_equal(a.faces, b.faces)
        assert np.abs(a.positions - b.positions).max() < 1e-15
    a, b = fx.uv_sphere(9, 8), ref.fixture(1, 9, 8, r=0.5)
    assert np.array_equal(a.faces, b.faces) and np.abs(a.positions - b.positions).max() < 1e-15
    a, b = fx.star_blob(4, 20, 20), ref.fixture(2, 20, 20, c=4, r=0.5)
    assert np.array_equal(a.faces, b.faces) and np.abs(a.positions - b.positions).max() < 1e-12
    assert np.array_equal(fx.random_points_in_box(50, (-1, -1, -1), (1, 1, 1), 31),
                          ref.random_points(50, (-1, -1, -1), (1, 1, 1), 31))
    assert np.abs(fx.random_unit_vectors(50, 22) - ref.random_units(50, 22)).max() < 1e-15


def test_reference_spatial_suite_passes_on_its_own_build(ref):
    exe = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "test_spatial")
    if not os.path.exists(exe):
        pytest.skip("reference test binary not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "14/14 test cases passed" in r.stdout


BAND_CASES = ("ico4", "plane", "torus", "domain")


def band_inputs(d, name):
    mesh = TriangleMesh(d[f"{name}_pos"], d[f"{name}_faces"])
    res, band, dil = d[f"{name}_params"]
    dom = d[f"{name}_domain"]
    return mesh, int(res), float(band), int(dil), (None if np.isnan(dom).any() else dom)


@pytest.mark.parametrize("case", BAND_CASES)
def test_port_matches_reference_golden_surface_band(port, case):
    """markSurfaceBand (signfield/sign_grid.cpp:23-69): labels, f32 distances
    and grid parameters bit-for-bit against the reference's own build."""
    d = load("band.npz")
    mesh, res, band, dil, dom = band_inputs(d, case)
    labels, dist, grid = port.surface_band(mesh, res, band, dil, dom)
    assert np.array_equal(labels, d[f"{case}_labels"])
    assert np.array_equal(u32(dist), u32(d[f"{case}_dist"]))
    assert np.array_equal(grid, d[f"{case}_grid"])


def test_port_surface_band_errors(port):
    from oracle.bindings import OracleError
    ico = TriangleMesh(load("band.npz")["domain_pos"], load("band.npz")["domain_faces"])
    for args, code in [((7, 1.0, 2, None), 12), ((32, 1.0, -1, None), 12), ((12, 1.0, 2, None), 12),
                       ((32, 1.0, 2, (0, 0, 0, 1, 1, 1)), 3)]:
        with pytest.raises(OracleError) as e:
            port.surface_band(ico, *args)
        assert e.value.code == code


VIEW_CASES = ("nested", "blob", "dup")


def f32bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.mark.parametrize("case", VIEW_CASES)
def test_port_matches_reference_golden_views(port, case):
    """renderView face/depth images and castVisibility hit histograms
    (render/raster.cpp:12-102, visibility/visibility.cpp:13-59) bit-for-bit."""
    d = load("views.npz")
    assert np.array_equal(port.fibonacci_cameras(8, 0.55), d["cams"])
    m = TriangleMesh(d[f"{case}_pos_in"], d[f"{case}_faces"])
    face, depth, pos, nrm = port.render_views(m, d["cams"], 96, d[f"{case}_vn"])
    assert np.array_equal(face, d[f"{case}_face"])
    assert np.array_equal(f32bits(depth), f32bits(d[f"{case}_depth"]))
    if case == "blob":
        assert np.array_equal(f32bits(pos[:2]), f32bits(d["blob_position"]))
        assert np.array_equal(f32bits(nrm[:2]), f32bits(d["blob_normal"]))
        cf, cd, _, _ = port.render_views(TriangleMesh(m.positions, np.ascontiguousarray(m.faces[:, ::-1])), d["cams"][:2], 96,
                                       d["blob_vn"], cull=True)
        assert np.array_equal(cf, d["blob_cull_face"])
        assert np.array_equal(f32bits(cd), f32bits(d["blob_cull_depth"]))
    assert np.array_equal(port.cast_visibility(m, 32, 96), d[f"{case}_hits"])


def test_reference_texfuse_reproduces_golden(ref):
    """The texfuse golden (tests/golden/texfuse.npz, make_golden.py) is
    reproducible from the reference build: fuse.cpp / mips.cpp are
    deterministic given the committed inputs."""
    d = np.load(os.path.join(GOLDEN, "texfuse.npz"))
    vres, diag = int(d["vres"]), float(d["diag"])
    for i in range(d["cams"].shape[0]):
        m = ref.edge_mask(d["v_pos"][i], d["v_face"][i], diag, 0.02)
        assert np.array_equal(m, d["masks"][i])
        chain, nm = ref.build_mips(d["colors"][i], 6, 0.2)
        assert np.array_equal(chain, d["chains"][i])
        c, s = ref.backproject_view(d["g_position"], d["g_valid"], 64, d["cams"][i], vres, 3, nm, chain, m)
        assert np.array_equal(c, d["parts"][i]) and np.array_equal(s, d["sampled"][i])
        inc = ref.incidence_map(d["g_position"], d["g_normal"], d["g_valid"], 64, d["cams"][i], vres, d["v_depth"][i],
                                diag, 0.005)
        assert np.array_equal(inc, d["incidence"][i])
    out, filled = ref.blend_views(d["parts"], d["sampled"], d["incidence"], d["priors"])
    assert np.array_equal(out, d["blend"]) and np.array_equal(filled, d["filled"])
    assert int(filled.sum()) > 0
