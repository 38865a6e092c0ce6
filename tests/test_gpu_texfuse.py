"""GPU parity of the texfuse G-buffer consumers against the
reference's own fuse.cpp / mips.cpp (compiled into oracle/_ref).

Bars:
  edgeMask, buildMips, incidenceMap, sampled / filled flags : bit-exact
  backprojectView, blendViews colours                        : within 1 f32 ulp
      (the footprint's log2 and the blend's log / exp are CUDA's, within 1 ulp
      of glibc's in f64; every other operation is the reference's expression)
"""
import numpy as np
import pytest

from paper_2605_26137_b200 import capi
from paper_2605_26137_b200 import fixtures as fx
from paper_2605_26137_b200 import meshforge as mf
from paper_2605_26137_b200 import texfuse as tf

pytestmark = pytest.mark.gpu

VRES = 128


def ulp_diff(a, b):
    a = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64)
    a = np.where(a < 0, -(a & 0x7fffffff), a)
    b = np.where(b < 0, -(b & 0x7fffffff), b)
    return np.abs(a - b)


@pytest.fixture(scope="module")
def scene(ref):
    p = fx.bake_pair(48, 8, 192, name="texfuse")
    g = mf.rasterize_gbuffer(p.lowpoly, p.res)
    cams = tf.standard_cameras(0.8)
    face, depth, pos, nrm = ref.render_views(p.dense, cams, VRES)
    # synthetic appearance: smooth colours of the world position (background 0)
    fg = (face >= 0)[..., None]
    col = np.concatenate([0.5 + 0.5 * np.sin(7.0 * pos[..., :1] + 1.0), 0.5 + 0.5 * np.cos(5.0 * pos[..., 1:2]),
                          0.5 + 0.5 * np.sin(3.0 * pos[..., 2:3] + pos[..., :1])], -1)
    col = (col * fg).astype(np.float32)
    return dict(p=p, g=g, cams=cams, face=face, depth=depth, pos=pos, col=col, diag=p.bbox_diagonal)


def test_edge_mask_bit_exact(gpu_ctx, ref, scene):
    for i in range(len(scene["cams"])):
        m = tf.edge_mask(scene["pos"][i], scene["face"][i], scene["diag"], 0.02)
        r = ref.edge_mask(scene["pos"][i], scene["face"][i], scene["diag"], 0.02)
        assert np.array_equal(m, r), i
        assert 0 < int(m.sum()) < m.size


@pytest.mark.parametrize("shape,levels,sharpen", [((VRES, VRES, 3), 6, 0.2), ((37, 53, 3), 8, 0.2),
                                                  ((40, 24, 1), 3, 0.0), ((5, 3, 2), 9, 0.5)])
def test_build_mips_bit_exact(gpu_ctx, ref, shape, levels, sharpen):
    rng = np.random.default_rng(5)
    base = rng.standard_normal(shape).astype(np.float32)
    chain = tf.build_mips(base, levels, sharpen)
    flat, n = ref.build_mips(base, levels, sharpen)
    assert len(chain) == n
    assert np.array_equal(np.concatenate([c.reshape(-1) for c in chain]), flat)
    assert np.array_equal(chain[0], base)


def test_incidence_map_bit_exact(gpu_ctx, ref, scene):
    g, n = scene["g"], scene["g"].resolution
    hits = 0
    for i, cam in enumerate(scene["cams"]):
        out = tf.incidence_map(g, cam, VRES, scene["depth"][i], scene["diag"], 0.005)
        r = ref.incidence_map(g.position, g.normal, g.valid, n, cam, VRES, scene["depth"][i], scene["diag"], 0.005)
        assert np.array_equal(out.reshape(-1).view(np.uint32), r.view(np.uint32)), i
        hits += int((r > 0).sum())
    assert hits > 0


def _ref_partials(ref, scene):
    g, n = scene["g"], scene["g"].resolution
    parts = []
    for i, cam in enumerate(scene["cams"]):
        mask = ref.edge_mask(scene["pos"][i], scene["face"][i], scene["diag"], 0.02)
        flat, nm = ref.build_mips(scene["col"][i], 6, 0.2)
        col, samp = ref.backproject_view(g.position, g.valid, n, cam, VRES, 3, nm, flat, mask)
        inc = ref.incidence_map(g.position, g.normal, g.valid, n, cam, VRES, scene["depth"][i], scene["diag"], 0.005)
        parts.append((mask, col, samp, inc))
    return parts


def test_backproject_view_matches_reference(gpu_ctx, ref, scene):
    g, n = scene["g"], scene["g"].resolution
    total = sampled = 0
    worst = 0
    for i, cam in enumerate(scene["cams"]):
        mask = ref.edge_mask(scene["pos"][i], scene["face"][i], scene["diag"], 0.02)
        mips = tf.build_mips(scene["col"][i], 6, 0.2)
        col, samp = tf.backproject_view(g, cam, VRES, mips, mask)
        flat, nm = ref.build_mips(scene["col"][i], 6, 0.2)
        rcol, rsamp = ref.backproject_view(g.position, g.valid, n, cam, VRES, 3, nm, flat, mask)
        assert np.array_equal(samp.reshape(-1), rsamp), i
        d = ulp_diff(col.reshape(-1), rcol.reshape(-1))
        worst = max(worst, int(d.max()))
        total += int((d != 0).sum())
        sampled += int(rsamp.sum())
    assert sampled > 1000
    assert worst <= 1, worst
    assert total <= max(1, sampled // 10000), total  # ulp-level differences stay exceptional


def test_blend_views_matches_reference(gpu_ctx, ref, scene):
    parts = _ref_partials(ref, scene)
    n = scene["g"].resolution
    cols = [c.reshape(n, n, 3) for _, c, _, _ in parts]
    samps = [s.reshape(n, n) for _, _, s, _ in parts]
    incs = [i.reshape(n, n) for _, _, _, i in parts]
    pri = tf.standard_view_priors()
    out, filled = tf.blend_views(cols, samps, incs, pri)
    rout, rfilled = ref.blend_views(np.stack([c.reshape(-1, 3) for c in cols]), np.stack([s.reshape(-1) for s in samps]),
                                    np.stack([i.reshape(-1) for i in incs]), pri)
    assert np.array_equal(filled.reshape(-1), rfilled)
    assert int(rfilled.sum()) > 1000
    assert ulp_diff(out.reshape(-1), rout.reshape(-1)).max() <= 1


def test_fuse_views_matches_reference_composition(gpu_ctx, ref, scene):
    g, n = scene["g"], scene["g"].resolution
    parts = _ref_partials(ref, scene)
    pri = tf.standard_view_priors()
    rout, rfilled = ref.blend_views(np.stack([c for _, c, _, _ in parts]), np.stack([s for _, _, s, _ in parts]),
                                    np.stack([i for _, _, _, i in parts]), pri)
    out, filled = tf.fuse_views(g, scene["cams"], VRES, scene["pos"], scene["face"], scene["depth"], scene["col"], pri,
                                scene["diag"])
    assert np.array_equal(filled.reshape(-1), rfilled)
    assert ulp_diff(out.reshape(-1), rout.reshape(-1)).max() <= 1
    # options: no sharpening, fewer mips, sharper incidence exponent
    o = tf.FuseOptions.defaults()
    assert o.mip_levels == 6 and abs(o.alpha - 4.0) < 1e-12
    o.sharpen_strength, o.mip_levels, o.alpha = 0.0, 3, 2.0
    out2, filled2 = tf.fuse_views(g, scene["cams"], VRES, scene["pos"], scene["face"], scene["depth"], scene["col"],
                                  pri, scene["diag"], options=o)
    assert np.array_equal(filled2, filled)
    assert not np.array_equal(out2, out)


def test_texfuse_errors(gpu_ctx, scene):
    g = scene["g"]
    with pytest.raises(capi.MeshforgeError) as e:
        tf.edge_mask(scene["pos"][0], scene["face"][0], 0.0)
    assert e.value.code == "InvalidConfig"
    with pytest.raises(capi.MeshforgeError) as e:
        tf.build_mips(scene["col"][0], 0)
    assert e.value.code == "InvalidConfig"
    with pytest.raises(capi.MeshforgeError) as e:
        tf.build_mips(scene["col"][0], 3, -1.0)
    assert e.value.code == "InvalidConfig"
    with pytest.raises(capi.MeshforgeError) as e:
        tf.incidence_map(g, scene["cams"][0], VRES, scene["depth"][0], scene["diag"], 0.0)
    assert e.value.code == "InvalidConfig"
    with pytest.raises(capi.MeshforgeError) as e:
        tf.incidence_map(g, scene["cams"][0], VRES, scene["depth"][0][:64], scene["diag"])
    assert e.value.code == "ShapeMismatch"
    with pytest.raises(capi.MeshforgeError) as e:
        tf.blend_views([], [], [], [])
    assert e.value.code == "InvalidConfig"
    one = np.zeros((4, 4, 3), np.float32)
    with pytest.raises(capi.MeshforgeError) as e:
        tf.blend_views([one], [np.ones((4, 4), np.uint8)], [np.ones((4, 4), np.float32)], [-1.0])
    assert e.value.code == "InvalidConfig"
    with pytest.raises(capi.MeshforgeError) as e:
        tf.fuse_views(g, scene["cams"][:0], VRES, scene["pos"], scene["face"], scene["depth"], scene["col"], [],
                      scene["diag"])
    assert e.value.code == "InvalidConfig"


def test_golden_texfuse(gpu_ctx):
    """The committed reference outputs (tests/golden/texfuse.npz), no _ref needed."""
    import os
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "texfuse.npz"))
    vres, diag = int(d["vres"]), float(d["diag"])
    g = mf.GBuffer.allocate(64)
    g.position[...] = d["g_position"].reshape(g.position.shape)
    g.normal[...] = d["g_normal"].reshape(g.normal.shape)
    g.valid[...] = d["g_valid"].reshape(g.valid.shape)
    for i in range(d["cams"].shape[0]):
        m = tf.edge_mask(d["v_pos"][i], d["v_face"][i], diag)
        assert np.array_equal(m, d["masks"][i])
        chain = tf.build_mips(d["colors"][i], 6, 0.2)
        assert np.array_equal(np.concatenate([c.reshape(-1) for c in chain]), d["chains"][i])
        col, samp = tf.backproject_view(g, d["cams"][i], vres, chain, m)
        assert np.array_equal(samp.reshape(-1), d["sampled"][i])
        assert ulp_diff(col.reshape(-1), d["parts"][i].reshape(-1)).max() <= 1
        inc = tf.incidence_map(g, d["cams"][i], vres, d["v_depth"][i], diag)
        assert np.array_equal(inc.reshape(-1), d["incidence"][i])
    out, filled = tf.fuse_views(g, d["cams"], vres, d["v_pos"], d["v_face"], d["v_depth"], d["colors"], d["priors"],
                                diag)
    assert np.array_equal(filled.reshape(-1), d["filled"])
    assert ulp_diff(out.reshape(-1), d["blend"].reshape(-1)).max() <= 1
