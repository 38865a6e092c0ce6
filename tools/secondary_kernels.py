"""One call of each secondary device path on config-B-sized
inputs, for ncu captures (tools/ncu_all.sh): raycastFirst / closestPointWithin
over 10^6 points, markSurfaceBand 256^3, castVisibility (64 views x 1024^2),
the API dilateSeams (sparse r=4, fused r=40), texfuse (fuseViews of 10 views
at 1024^2 onto the 2048^2 G-buffer)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_26137_b200 import capi, fixtures as fx, meshforge as mf  # noqa: E402
import bench  # noqa: E402

p = fx.config_pair("B")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)  # the context launches on it (the default stream would be NULL)
ctx = capi.Context(0, stream.cuda_stream)
lo = capi.DeviceMesh(ctx, p.lowpoly)
hi = capi.DeviceMesh(ctx, p.dense)
bvh = mf.Bvh(p.dense, ctx=ctx)
rng = np.random.default_rng(3)
q = rng.uniform(p.dense.positions.min(0), p.dense.positions.max(0), (1 << 20, 3))
d = rng.standard_normal((1 << 20, 3))
d /= np.linalg.norm(d, axis=1, keepdims=True)
bvh.raycasts(q, d)
bvh.closest_points(q, p.max_distance_fraction * p.bbox_diagonal)
bvh.surface_band(256, 1.0, 2)
hits = np.zeros(p.dense.face_count(), np.int64)
mv = p.dense.view()
capi.check(ctx.lib.mf_cast_visibility(ctx.h, ctypes.byref(mv), 8, 1024, hits.ctypes.data_as(ctypes.c_void_p), None))
res = 24
field = np.linspace(-1.0, 1.0, res ** 3, dtype=np.float32)
bvh.sample_sdf(res, p.dense.positions.min(0) - 0.05, 1.3 / res, field, q[: 1 << 18])
g = mf.rasterize_gbuffer(p.lowpoly, p.res)
img = rng.integers(0, 255, (p.res, p.res, 3), dtype=np.uint8)
mf.dilate_seams(img, g, 4)
mf.dilate_seams(img, g, 40)
# texfuse: one fuseViews call (10 views at 1024^2 onto the 2048^2 G-buffer)
bench.texfuse_bench(ctx, lo, p, 1, once=True)
torch.cuda.synchronize()
print("secondary kernels done")
