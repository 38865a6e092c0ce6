"""GPU: row-slab bakes (the multi-GPU partition of SURVEY §8e, run here as
sequential shards on one device) reproduce the full bake exactly, and the
coverage pre-pass matches the oracle's per-row valid counts."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2605_26137_b200 import capi, sharding
from paper_2605_26137_b200 import fixtures as fx

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [2, 3, 5])
def test_row_slabs_reassemble_the_full_bake(gpu_ctx, port, k):
    p = fx.bake_pair(64, 8, 256, name="slabs")
    ctx = capi.Context(0, torch.cuda.current_stream().cuda_stream)
    lo, hi = capi.DeviceMesh(ctx, p.lowpoly), capi.DeviceMesh(ctx, p.dense)
    rows = np.zeros(p.res, np.int64)
    capi.check(ctx.lib.mf_coverage_rows(ctx.h, lo.h, p.res, ctypes.c_void_p(rows.ctypes.data)))
    g = port.raster_gbuffer(p.lowpoly, p.res)
    assert np.array_equal(rows, g.valid.reshape(p.res, p.res).sum(1))
    full = torch.empty((p.res, p.res, 3), dtype=torch.uint8, device="cuda")
    capi.check(ctx.lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, p.res, p.bbox_diagonal, p.max_distance_fraction,
                                              4, 0, p.res, full.data_ptr(), None))
    parts = []
    for b, e in sharding.balanced_row_ranges(rows, k):
        slab = torch.empty((e - b, p.res, 3), dtype=torch.uint8, device="cuda")
        capi.check(ctx.lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, p.res, p.bbox_diagonal,
                                                  p.max_distance_fraction, 4, b, e, slab.data_ptr(), None))
        parts.append(slab)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, 0), full)
    ref = port.bake(p.lowpoly, p.dense, p.res, p.bbox_diagonal, p.max_distance_fraction, 4)
    d = np.abs(full.cpu().numpy().reshape(-1, 3).astype(int) - ref["rgb"].astype(int))
    assert d.max() <= 1
