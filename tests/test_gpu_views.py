"""GPU: ortho pixel-ray views through the LBVH:
renderView (render/raster.cpp:12-102) images and castVisibility
(visibility/visibility.cpp:13-59) hit histograms, bit-exact against the
reference's goldens and the C restatement (oracle/mf_oracle.c)."""
import os

import numpy as np
import pytest

from paper_2605_26137_b200 import fixtures as fx
from paper_2605_26137_b200 import meshforge as mf
from paper_2605_26137_b200.mesh import TriangleMesh

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def f32bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def test_fibonacci_cameras_match_reference(gpu_ctx):
    d = np.load(os.path.join(GOLDEN, "views.npz"))
    assert np.array_equal(mf.fibonacci_cameras(8, 0.55), d["cams"])


@pytest.mark.parametrize("case", ["nested", "blob", "dup"])
def test_render_views_match_reference_golden(gpu_ctx, case):
    d = np.load(os.path.join(GOLDEN, "views.npz"))
    m = TriangleMesh(d[f"{case}_pos_in"], d[f"{case}_faces"])
    face, depth, pos, nrm = mf.render_views(m, d["cams"], 96, d[f"{case}_vn"])
    assert np.array_equal(face, d[f"{case}_face"])
    assert np.array_equal(f32bits(depth), f32bits(d[f"{case}_depth"]))
    if case == "blob":
        assert np.array_equal(f32bits(pos[:2]), f32bits(d["blob_position"]))
        assert np.array_equal(f32bits(nrm[:2]), f32bits(d["blob_normal"]))
        cf, cd, _, _ = mf.render_views(TriangleMesh(m.positions, np.ascontiguousarray(m.faces[:, ::-1])), d["cams"][:2], 96,
                                     d["blob_vn"], backface_cull=True)
        assert np.array_equal(cf, d["blob_cull_face"])
        assert np.array_equal(f32bits(cd), f32bits(d["blob_cull_depth"]))


@pytest.mark.parametrize("case", ["nested", "blob", "dup"])
def test_cast_visibility_matches_reference_golden(gpu_ctx, case):
    d = np.load(os.path.join(GOLDEN, "views.npz"))
    m = TriangleMesh(d[f"{case}_pos_in"], d[f"{case}_faces"])
    hits, state = mf.cast_visibility(m, 32, 96)
    assert np.array_equal(hits, d[f"{case}_hits"])
    assert np.array_equal(state, (d[f"{case}_hits"] > 0).astype(np.uint8))


def test_sealed_inner_sphere_collects_no_hits(gpu_ctx):
    """test_visibility.cpp:138-147: the inner shell of nested spheres is never hit."""
    d = np.load(os.path.join(GOLDEN, "views.npz"))
    m = TriangleMesh(d["nested_pos_in"], d["nested_faces"])
    hits, state = mf.cast_visibility(m, 64, 256)
    outer = 20 * 4 ** 3  # icosphere(3)
    assert hits[outer:].sum() == 0 and state[outer:].sum() == 0
    assert state[:outer].all()


def test_cast_visibility_dense_blob_matches_port(gpu_ctx, port):
    """A config-A dense mesh (200k faces), 12 views x 192^2, vs the oracle."""
    m = fx.config_pair("A").dense
    hits, _ = mf.cast_visibility(m, 12, 192)
    assert np.array_equal(hits, port.cast_visibility(m, 12, 192))
    assert hits.sum() > 0


def test_cast_visibility_errors(gpu_ctx):
    from paper_2605_26137_b200.capi import MeshforgeError
    tri = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    hits, state = mf.cast_visibility(tri, 16, 64)  # test_visibility.cpp:107-114
    assert state[0] == 1 and hits[0] >= 1
    for vp, res in ((0, 64), (16, 0)):
        with pytest.raises(MeshforgeError) as e:
            mf.cast_visibility(tri, vp, res)
        assert e.value.status == 12
    with pytest.raises(MeshforgeError) as e:
        mf.cast_visibility(TriangleMesh(np.zeros((3, 3)), np.zeros((0, 3), np.int32)), 16, 64)
    assert e.value.status == 1
