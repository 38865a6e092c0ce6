"""GPU: the fused bake's optional atlas encodings (north_star item 4,
mf_bake_normal_map_ex / _dev_ex).

  RGBA8 : the RGB8 atlas byte for byte plus alpha 255 (host and device paths,
          full atlas with the dilation links and row slabs with the dilation pass)
  RG16  : unorm16 of the oracle's pre-quantisation tangent-space x, y within one
          code (q = round((v + 1) / 2 * 65535); GPU and oracle ts differ by
          acos ulps only), (32768, 32768) for background / neutral texels, and
          every dilated texel equal to its source (the oracle's dilateSeams run
          over the 4-byte pixels)
"""
import ctypes

import numpy as np
import pytest
import torch

from paper_2605_26137_b200 import capi
from paper_2605_26137_b200 import fixtures as fx
from paper_2605_26137_b200 import meshforge as mf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair():
    return fx.bake_pair(64, 8, 256, name="formats")


def _enc16(v):
    q = np.rint((v + 1.0) * 0.5 * 65535.0)  # llround ties away; exact .5 never occurs for these ts
    return np.clip(q, 0, 65535).astype(np.int64)


@pytest.mark.parametrize("radius", [0, 4, 40])
def test_rgba8_is_rgb8_plus_alpha(gpu_ctx, pair, radius):
    p = pair
    rgb = mf.bake_normal_map(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, radius)
    rgba = mf.bake_normal_map_ex(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, radius,
                                 fmt=mf.ATLAS_RGBA8)
    assert rgba.shape == (p.res, p.res, 4)
    assert np.array_equal(rgba[..., :3], rgb)
    assert (rgba[..., 3] == 255).all()
    # the RGB8 format through the _ex entry is mf_bake_normal_map
    rgb2 = mf.bake_normal_map_ex(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, radius,
                                 fmt=mf.ATLAS_RGB8)
    assert np.array_equal(rgb2, rgb)


def _expected_rg16(port, p, radius):
    ref = port.bake(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 0, debug=True)
    face, ts = ref["face"].reshape(-1), ref["ts"].reshape(-1, 3)
    g = port.raster_gbuffer(p.lowpoly, p.res)
    px = np.full((p.res * p.res, 2), 32768, np.int64)
    hit = face >= 0
    enc = _enc16(ts)
    nz = hit & (np.abs(ts).sum(1) > 0)
    px[nz, 0] = enc[nz, 0]
    px[nz, 1] = enc[nz, 1]
    raw = px.astype(np.uint16).view(np.uint8).reshape(p.res, p.res, 4).copy()
    out = port.dilate_seams(raw, p.res, p.res, 4, p.res, g.valid, radius)
    return np.asarray(out).reshape(p.res, p.res, 4).view(np.uint16).reshape(p.res, p.res, 2), ts, g.valid


@pytest.mark.parametrize("radius", [0, 4])
def test_rg16_matches_oracle_ts(gpu_ctx, port, pair, radius):
    p = pair
    rg = mf.bake_normal_map_ex(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, radius,
                               fmt=mf.ATLAS_RG16)
    assert rg.shape == (p.res, p.res, 2) and rg.dtype == np.uint16
    exp, ts, valid = _expected_rg16(port, p, radius)
    d = np.abs(rg.astype(np.int64) - exp.astype(np.int64))
    assert d.max() <= 1
    # a one-code difference only where the oracle value sits at a rounding boundary
    v = (ts[:, :2] + 1.0) * 0.5 * 65535.0
    edge = np.abs(v - np.floor(v) - 0.5) <= 1e-6
    bad = (d.reshape(-1, 2) == 1) & (valid.reshape(-1, 1) != 0)
    assert (edge[bad]).all()
    # decode round trip within the quantisation
    dec = mf.decode_rg16(rg).reshape(-1, 3)
    m = (valid.reshape(-1) != 0) & (np.abs(ts).sum(1) > 0)
    assert np.abs(dec[m, :2] - ts[m, :2]).max() <= 1.0 / 65535 + 1e-9


@pytest.mark.parametrize("fmt", [1, 2])
def test_dev_slabs_in_4byte_formats(gpu_ctx, pair, fmt):
    """Row slabs (dilation pass over 4-byte pixels) reassemble the full atlas."""
    p = pair
    ctx = capi.Context(0, torch.cuda.current_stream().cuda_stream)
    lo, hi = capi.DeviceMesh(ctx, p.lowpoly), capi.DeviceMesh(ctx, p.dense)
    full = torch.empty((p.res, p.res, 4), dtype=torch.uint8, device="cuda")
    capi.check(ctx.lib.mf_bake_normal_map_dev_ex(ctx.h, lo.h, hi.h, p.res, p.bbox_diagonal,
                                                 p.max_distance_fraction, 4, 0, p.res, fmt, full.data_ptr(), None))
    parts = []
    for b, e in ((0, 77), (77, 180), (180, p.res)):
        slab = torch.empty((e - b, p.res, 4), dtype=torch.uint8, device="cuda")
        capi.check(ctx.lib.mf_bake_normal_map_dev_ex(ctx.h, lo.h, hi.h, p.res, p.bbox_diagonal,
                                                     p.max_distance_fraction, 4, b, e, fmt, slab.data_ptr(), None))
        parts.append(slab)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, 0), full)
    host = mf.bake_normal_map_ex(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 4, fmt=fmt)
    assert np.array_equal(full.cpu().numpy().reshape(-1), host.reshape(-1).view(np.uint8))


def test_format_errors(gpu_ctx, pair):
    p = pair
    with pytest.raises(capi.MeshforgeError) as e:
        mf.bake_normal_map_ex(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 4, fmt=7,
                              out=np.zeros((p.res, p.res, 4), np.uint8))
    assert e.value.status == -3
    ctx = capi.Context(0, torch.cuda.current_stream().cuda_stream)
    lo, hi = capi.DeviceMesh(ctx, p.lowpoly), capi.DeviceMesh(ctx, p.dense)
    buf = torch.empty(p.res * p.res * 4 + 4, dtype=torch.uint8, device="cuda")
    rc = ctx.lib.mf_bake_normal_map_dev_ex(ctx.h, lo.h, hi.h, p.res, p.bbox_diagonal, p.max_distance_fraction, 4, 0,
                                           p.res, 2, ctypes.c_void_p(buf.data_ptr() + 1), None)
    assert rc == -3  # misaligned 4-byte atlas
