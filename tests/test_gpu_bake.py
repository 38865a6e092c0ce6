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
