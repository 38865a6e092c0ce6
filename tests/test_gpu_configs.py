"""GPU: parity at BASELINE.json sizes against the CPU oracle (all host cores).

Config B (1,003,520-face dense, 2048^2): every texel - hit faces bit-exact,
ts within 1e-3 / 0.1 deg, RGB within the boundary rule. Config E's dense mesh
(3,996,180 faces, lowpoly offset x1.04, maxDistanceFraction 0.05 - the deep,
divergent traversal) at a 1024^2 atlas to keep the oracle's run short."""
import numpy as np
import pytest

from paper_2605_26137_b200 import fixtures as fx
from paper_2605_26137_b200 import meshforge as mf

from test_gpu_bake import ANG_TOL_DEG, TS_TOL, assert_rgb_parity

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def check_pair(p, port):
    out = mf.bake_normal_map(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 4, debug=True,
                             stats=True)
    o = port.bake(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 4, debug=True)
    assert np.array_equal(out["face"], o["face"])
    hit = o["face"] >= 0
    assert np.abs(out["ts"] - o["ts"]).max() <= TS_TOL
    cosang = np.clip((out["ts"][hit] * o["ts"][hit]).sum(1), -1, 1)
    assert np.degrees(np.arccos(cosang)).max() <= ANG_TOL_DEG
    assert_rgb_parity(out["rgb"], o["rgb"], o["ts"])
    assert out["stats"]["valid_texels"] == o["n_valid"] and out["stats"]["queries"] == o["n_queries"]
    return out, o


def test_config_b_full_parity(gpu_ctx, port):
    out, o = check_pair(fx.config_pair("B"), port)
    assert o["n_valid"] > 2_500_000


def test_config_e_mesh_deep_traversal_parity(gpu_ctx, port):
    c = fx.CONFIGS["E"]
    p = fx.bake_pair(c["n_dense"], c["n_low"], 1024, c["frac"], c["seed"], c["low_scale"], name="E1024")
    assert p.dense.face_count() == 3_996_180
    out, o = check_pair(p, port)
    assert (o["face"] >= 0).sum() > 500_000
