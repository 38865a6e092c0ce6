"""GPU parity: the CUDA bake path (through the C ABI) vs the CPU oracle.

Bars (SURVEY §8c parity table, BASELINE north_star tolerance):
  valid / reliable masks, positions, hit-face ids, dilation : bit-exact
  normal                                                    : bit-exact (no acos on its path)
  tangent / bitangent                                       : |d| <= 1e-6 (CUDA acos vs glibc acos)
  pre-quantisation ts                                       : <= 1e-3 per component and <= 0.1 deg
  RGB8                                                      : identical, except +-1 LSB where the
                                                              oracle's (v+1)*127.5 is within 1e-3*127.5
                                                              of a .5 rounding boundary
"""
import numpy as np
import pytest

from paper_2605_26137_b200 import fixtures as fx
from paper_2605_26137_b200 import meshforge as mf

pytestmark = pytest.mark.gpu

TS_TOL = 1e-3
ANG_TOL_DEG = 0.1


@pytest.fixture(scope="module")
def pair_a():
    return fx.config_pair("A")


def _u32(a):
    return np.ascontiguousarray(a).view(np.uint32)


def assert_rgb_parity(rgb, rgb_ref, ts_ref):
    rgb = rgb.reshape(-1, 3).astype(np.int32)
    rgb_ref = rgb_ref.reshape(-1, 3).astype(np.int32)
    diff = np.abs(rgb - rgb_ref)
    assert diff.max() <= 1
    if diff.max() == 1:
        # only where the oracle value sits within the tolerance of a .5 boundary
        bad = np.argwhere(diff == 1)
        v = (ts_ref.reshape(-1, 3)[bad[:, 0], bad[:, 1]] + 1.0) * 127.5
        frac = np.abs(v - np.floor(v) - 0.5)
        assert (frac <= TS_TOL * 127.5).all()


def test_raster_gbuffer_matches_oracle(gpu_ctx, port, pair_a):
    lo, res = pair_a.lowpoly, pair_a.res
    g = mf.rasterize_gbuffer(lo, res)
    o = port.raster_gbuffer(lo, res)
    assert np.array_equal(g.valid, o.valid)
    assert np.array_equal(g.reliable, o.reliable)
    assert int(g.valid.sum()) > 0.5 * res * res
    assert np.array_equal(_u32(g.position), _u32(o.position))
    assert np.array_equal(_u32(g.normal), _u32(o.normal))
    assert np.abs(g.tangent - o.tangent).max() <= 1e-6
    assert np.abs(g.bitangent - o.bitangent).max() <= 1e-6


def test_fused_bake_matches_oracle(gpu_ctx, port, pair_a):
    p = pair_a
    out = mf.bake_normal_map(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 4,
                             debug=True, stats=True)
    o = port.bake(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 4, debug=True)
    # hit / miss / unreliable / invalid classification and hit-face ids: bit-exact
    assert np.array_equal(out["face"], o["face"])
    hit = o["face"] >= 0
    assert hit.sum() > 0
    dts = np.abs(out["ts"] - o["ts"]).max()
    assert dts <= TS_TOL
    cosang = np.clip((out["ts"][hit] * o["ts"][hit]).sum(1), -1, 1)
    assert np.degrees(np.arccos(cosang)).max() <= ANG_TOL_DEG
    assert_rgb_parity(out["rgb"], o["rgb"], o["ts"])
    st = out["stats"]
    assert st["valid_texels"] == o["n_valid"]
    assert st["queries"] == o["n_queries"]


def test_transfer_normals_on_identical_gbuffer(gpu_ctx, port, pair_a):
    p = pair_a
    g = port.raster_gbuffer(p.lowpoly, p.res)
    gb = mf.GBuffer(p.res, g.position, g.normal, g.tangent, g.bitangent, g.valid, g.reliable)
    rgb = mf.transfer_normals(gb, p.dense, p.bbox_diagonal, p.max_distance_fraction)
    rgb_o, face_o, ts_o = port.transfer_normals(g, p.dense, p.bbox_diagonal, p.max_distance_fraction, debug=True)
    assert_rgb_parity(rgb, rgb_o, ts_o)


@pytest.mark.parametrize("radius", [0, 1, 2, 4, 7, 40])
def test_dilate_seams_bit_exact(gpu_ctx, port, radius):
    rng = np.random.default_rng(radius)
    res = 97
    valid = (rng.random(res * res) < 0.03).astype(np.uint8)
    img = rng.integers(0, 256, (res, res, 3), dtype=np.uint8)
    g = mf.GBuffer.allocate(res)
    g.valid[:] = valid
    out = mf.dilate_seams(img, g, radius)
    ref = port.dilate_seams(img.reshape(-1, 3), res, res, 3, res, valid, radius).reshape(res, res, 3)
    assert np.array_equal(out, ref)


# ---------------------------------------------------------------- reference goldens
import os  # noqa: E402

from paper_2605_26137_b200.mesh import TriangleMesh  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("case", ["tiny", "small", "cage"])
def test_gpu_matches_reference_golden_bake(gpu_ctx, case):
    """Against outputs of the reference's own code (tests/golden/make_golden.py)."""
    d = np.load(os.path.join(GOLDEN, f"bake_{case}.npz"))
    p = fx.bake_pair(int(d["n_dense"]), int(d["n_low"]), int(d["res"]), float(d["frac"]), int(d["seed"]),
                     float(d["low_scale"]), name=case)
    g = mf.rasterize_gbuffer(p.lowpoly, p.res)
    assert np.array_equal(g.valid, d["valid"]) and np.array_equal(g.reliable, d["reliable"])
    assert np.array_equal(_u32(g.position), _u32(d["position"]))
    assert np.array_equal(_u32(g.normal), _u32(d["normal"]))
    assert np.abs(g.tangent - d["tangent"]).max() <= 1e-6
    out = mf.bake_normal_map(p.lowpoly, p.dense, p.res, p.bbox_diagonal, float(d["frac"]), 4, debug=True)
    assert np.array_equal(out["face"], d["face"])
    assert np.abs(out["ts"] - d["ts"]).max() <= TS_TOL
    assert_rgb_parity(out["rgb"], d["rgb"], d["ts"])


def test_gpu_reference_kats(gpu_ctx):
    """test_bake.cpp:77-200,253-274 known answers, through the Python mirror API."""
    d = np.load(os.path.join(GOLDEN, "kats.npz"))
    m = TriangleMesh([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [1, 0, 200]], [[0, 1, 2], [0, 2, 3], [1, 4, 2]],
                     uvs=[[0.05, 0.05], [0.35, 0.05], [0.35, 0.35], [0.05, 0.35], [0.65, 0.05]],
                     face_uvs=[[0, 1, 2], [0, 2, 3], [1, 4, 2]])
    g = mf.rasterize_gbuffer(m, 128)
    assert np.array_equal(g.valid, d["od_valid"]) and np.array_equal(g.reliable, d["od_reliable"])
    assert np.array_equal(mf.transfer_normals(g, m, m.bbox_diagonal()).reshape(-1, 3), d["od_rgb"])
    q, far = fx.identity_quad(), fx.identity_quad()
    far.positions[:, 2] += 0.08
    g = mf.rasterize_gbuffer(q, 32)
    assert np.array_equal(mf.transfer_normals(g, far, float(np.sqrt(2.0))).reshape(-1, 3), d["far_rgb"])
    assert np.array_equal(mf.rasterize_gbuffer(q, 8).valid, d["fill_valid"])
    tri = TriangleMesh([[0, 0, 0], [2, 0, 0], [0, 2, 0]], [[0, 1, 2]], uvs=[[0, 0], [2, 0], [0, 2]],
                       face_uvs=[[0, 1, 2]])
    g = mf.rasterize_gbuffer(tri, 32)
    assert (g.valid == 1).all()
    assert np.array_equal(_u32(g.position), _u32(d["tri_position"]))
    gl = mf.GBuffer.allocate(11)
    gl.valid[:] = d["lone_valid"]
    out = mf.dilate_seams(d["lone_in"].reshape(11, 11, 3), gl, 2)
    assert np.array_equal(out.reshape(-1, 3), d["lone_out"])


def test_gpu_error_codes(gpu_ctx):
    """test_bake.cpp:126-133,332-350: same codes through the C ABI."""
    def code(fn):
        with pytest.raises(mf.MeshforgeError) as e:
            fn()
        return e.value.code

    bare = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    assert code(lambda: mf.rasterize_gbuffer(bare, 64)) == "InvalidGeometry"
    assert code(lambda: mf.rasterize_gbuffer(fx.identity_quad(), 0)) == "InvalidConfig"
    assert code(lambda: mf.rasterize_gbuffer(TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3))), 64)) == "EmptyMesh"
    overlap = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [0, 1, 1]],
                           [[0, 1, 2], [3, 4, 5]],
                           uvs=[[0.1, 0.1], [0.9, 0.1], [0.1, 0.9], [0.2, 0.2], [0.8, 0.2], [0.2, 0.8]],
                           face_uvs=[[0, 1, 2], [3, 4, 5]])
    assert code(lambda: mf.rasterize_gbuffer(overlap, 64)) == "AtlasOverlap"
    assert code(lambda: mf.bake_normal_map(overlap, fx.identity_quad(), 64, 1.0)) == "AtlasOverlap"
    g = mf.rasterize_gbuffer(fx.identity_quad(), 16)
    assert code(lambda: mf.transfer_normals(mf.GBuffer.allocate(0), fx.identity_quad(), 1.0)) == "InvalidConfig"
    assert code(lambda: mf.transfer_normals(g, fx.identity_quad(), 0.0)) == "InvalidConfig"
    empty = TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3)))
    assert code(lambda: mf.transfer_normals(g, empty, 1.0)) == "EmptyMesh"
    nan = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, np.nan, 0]], [[0, 1, 2]])
    assert code(lambda: mf.transfer_normals(g, nan, 1.0)) == "InvalidGeometry"
    assert code(lambda: mf.dilate_seams(np.zeros((8, 8, 3), np.uint8), g, 2)) == "ShapeMismatch"
    assert code(lambda: mf.dilate_seams(np.zeros((16, 16, 3), np.uint8), g, -1)) == "InvalidConfig"
    # the context survives errors
    assert mf.rasterize_gbuffer(fx.identity_quad(), 8).valid.sum() == 64


def test_gpu_wedge_tangents_and_vertex_normals(gpu_ctx):
    d = np.load(os.path.join(GOLDEN, "tangents.npz"))
    m = TriangleMesh(d["pos"], d["faces"], uvs=d["uvs"], face_uvs=d["face_uvs"])
    frames = mf.compute_wedge_tangents(m)
    # normals are exact; tangents/bitangents go through acos (CUDA vs glibc ulps)
    assert np.array_equal(frames[:, :, 2], d["frames"][:, :, 2])
    assert np.abs(frames - d["frames"]).max() <= 1e-12
    vm = TriangleMesh(d["vn_mesh_pos"], d["vn_mesh_faces"])
    assert np.array_equal(mf.compute_vertex_normals(vm), d["vnormals"])


def test_host_bake_error_order(gpu_ctx):
    """mf_bake_normal_map overlaps the dense upload with the lowpoly raster;
    its errors keep the reference composition's order (test_bake.cpp:205-206):
    lowpoly checks (gbuffer.cpp:93-97) -> AtlasOverlap (:157-159) ->
    transferNormals' checks (:195-199) -> dilateSeams' radius (:255)."""
    def code(fn):
        with pytest.raises(mf.MeshforgeError) as e:
            fn()
        return e.value.code

    quad = fx.identity_quad()
    bare = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    nan = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, np.nan, 0]], [[0, 1, 2]])
    oob = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 7]])
    empty = TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3)))
    overlap = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [0, 1, 1]],
                           [[0, 1, 2], [3, 4, 5]],
                           uvs=[[0.1, 0.1], [0.9, 0.1], [0.1, 0.9], [0.2, 0.2], [0.8, 0.2], [0.2, 0.8]],
                           face_uvs=[[0, 1, 2], [3, 4, 5]])
    assert code(lambda: mf.bake_normal_map(bare, nan, 32, 1.0)) == "InvalidGeometry"  # lowpoly first
    assert code(lambda: mf.bake_normal_map(quad, nan, 0, 1.0)) == "InvalidConfig"  # res before the dense mesh
    assert code(lambda: mf.bake_normal_map(overlap, nan, 32, 1.0)) == "AtlasOverlap"
    assert code(lambda: mf.bake_normal_map(overlap, quad, 32, 0.0)) == "AtlasOverlap"
    assert code(lambda: mf.bake_normal_map(quad, nan, 32, 1.0)) == "InvalidGeometry"
    assert code(lambda: mf.bake_normal_map(quad, oob, 32, 1.0)) == "InvalidGeometry"
    assert code(lambda: mf.bake_normal_map(quad, empty, 32, 1.0)) == "EmptyMesh"
    assert code(lambda: mf.bake_normal_map(quad, nan, 32, 0.0)) == "InvalidGeometry"  # mesh before config
    assert code(lambda: mf.bake_normal_map(quad, quad, 32, 0.0)) == "InvalidConfig"
    assert code(lambda: mf.bake_normal_map(quad, quad, 32, 1.0, radius=-1)) == "InvalidConfig"
    # and the context still bakes afterwards
    out = mf.bake_normal_map(quad, quad, 32, float(np.sqrt(2.0)))
    assert out.shape[:2] == (32, 32) or out.size == 32 * 32 * 3


@pytest.mark.parametrize("res,radius", [(None, 4), (None, 1), (None, 20), (300, 4), (100, 0), (64, 17)])
def test_host_bake_pinned_banded_download(gpu_ctx, port, pair_a, res, radius):
    """Host-buffer bake into pinned memory: the atlas is downloaded in row bands
    while the transfer runs (BandSync, cuStreamWaitValue32) and the dilation is
    resolved before the transfer (dilate_links). Byte-identical to the eager
    device path, and within the parity bar of the oracle."""
    torch = pytest.importorskip("torch")
    import os
    os.environ["MFB_BAND_CHECK"] = "1"  # every band signalled by the transfer's counts
    p = pair_a
    res = res or p.res
    pinned = torch.empty((res, res, 3), dtype=torch.uint8).pin_memory().numpy()
    pinned[:] = 7  # stale bytes must all be overwritten
    for _ in range(3):  # eager, captured, replayed graphs
        got = mf.bake_normal_map(p.lowpoly, p.dense, res, p.bbox_diagonal, p.max_distance_fraction, radius,
                                 out=pinned)
        ref = mf.bake_normal_map(p.lowpoly, p.dense, res, p.bbox_diagonal, p.max_distance_fraction, radius,
                                 debug=True)
        assert np.array_equal(got, ref["rgb"])
    o = port.bake(p.lowpoly, p.dense, res, p.bbox_diagonal, p.max_distance_fraction, radius, debug=True)
    assert_rgb_parity(pinned, o["rgb"], o["ts"])


def test_fused_bake_unreliable_faces(gpu_ctx, port):
    """Late reliability in the fused bake: the coverage kernel compacts every
    valid texel and the texels of unreliable faces (the stretched face of the
    test_bake.cpp:77-100 KAT) become dead records encoded as (128,128,255) by
    the transfer, dilated like any other source - equal to the port, through
    the device-mesh and the host-buffer (pinned and pageable) entry points."""
    torch = pytest.importorskip("torch")
    m = TriangleMesh([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [1, 0, 200]], [[0, 1, 2], [0, 2, 3], [1, 4, 2]],
                     uvs=[[0.05, 0.05], [0.35, 0.05], [0.35, 0.35], [0.05, 0.35], [0.65, 0.05]],
                     face_uvs=[[0, 1, 2], [0, 2, 3], [1, 4, 2]])
    dense = fx.bake_pair(24, 4, 64, name="unrel").dense
    dense.positions[:] = dense.positions * 250.0 + np.array([0.5, 0.5, 100.0])
    for radius in (0, 4, 9):
        o = port.bake(m, dense, 128, float(dense.bbox_diagonal()), 0.5, radius, debug=True)
        assert (o["face"] == -2).sum() > 0  # unreliable texels present
        out = mf.bake_normal_map(m, dense, 128, float(dense.bbox_diagonal()), 0.5, radius, debug=True, stats=True)
        assert np.array_equal(out["face"], o["face"])
        assert_rgb_parity(out["rgb"], o["rgb"], o["ts"])
        assert out["stats"]["queries"] == o["n_queries"]
        assert out["stats"]["valid_texels"] == o["n_valid"]
        for pinned in (True, False):
            buf = torch.empty((128, 128, 3), dtype=torch.uint8)
            if pinned:
                buf = buf.pin_memory()
            host = buf.numpy()
            for _ in range(3):  # eager, captured, replayed
                got = mf.bake_normal_map(m, dense, 128, float(dense.bbox_diagonal()), 0.5, radius, out=host)
                assert np.array_equal(got.reshape(-1, 3), out["rgb"].reshape(-1, 3))


@pytest.mark.parametrize("valence", [5, 16, 17, 40, 300])
def test_vertex_normals_high_valence_fans(gpu_ctx, port, valence):
    """computeVertexNormals (mesh.cpp:24-35) on a cone fan whose apex has the
    given valence (per-vertex slots hold 16 corners; more spill to the
    overflow list), plus a degenerate face naming one vertex twice: bit-exact
    vs the port (face-order sums)."""
    from paper_2605_26137_b200.mesh import TriangleMesh
    rng = np.random.default_rng(valence)
    ang = np.sort(rng.uniform(0, 2 * np.pi, valence))
    rim = np.stack([np.cos(ang), np.sin(ang), 0.1 * rng.standard_normal(valence)], 1)
    pos = np.vstack([[0.0, 0.0, 0.7], rim, [[0.3, 0.2, -0.4]]])
    faces = [[0, 1 + i, 1 + (i + 1) % valence] for i in range(valence)]
    faces.append([1, 1, valence + 1])  # degenerate: vertex 1 twice
    perm = rng.permutation(len(faces))  # apex corners spread over the face order
    m = TriangleMesh(pos, np.asarray(faces, np.int32)[perm])
    assert np.array_equal(mf.compute_vertex_normals(m), port.vertex_normals(m))
