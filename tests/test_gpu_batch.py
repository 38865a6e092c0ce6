"""GPU: several independent assets baked concurrently (SURVEY §8e config D
style: one mf_ctx + stream per asset, one host thread each) give exactly the
bytes the same assets give when baked one after another on one context.

Covers the ABI's threading contract (include/mfbake.h: distinct contexts may
be used from distinct threads concurrently) including the per-context CUDA
graph capture (second identical call) racing with eager first calls."""
import concurrent.futures as cf
import ctypes

import numpy as np
import pytest

from paper_2605_26137_b200 import capi
from paper_2605_26137_b200 import fixtures as fx

pytestmark = pytest.mark.gpu


def _bake(ctx, lo, hi, p, out):
    capi.check(ctx.lib.mf_bake_normal_map(ctx.h, ctypes.byref(lo), ctypes.byref(hi), p.res, p.bbox_diagonal,
                                          p.max_distance_fraction, 4, ctypes.c_void_p(out.ctypes.data), None, None,
                                          None))


def test_concurrent_contexts_match_serial(gpu_ctx):
    pairs = [fx.bake_pair(30 + 4 * i, 6 + i, 192 + 32 * i, seed=100 + i, name=f"batch{i}") for i in range(4)]
    views = [(p.lowpoly.view(), p.dense.view()) for p in pairs]
    serial = []
    for p, (lo, hi) in zip(pairs, views):
        out = np.zeros((p.res, p.res, 3), np.uint8)
        _bake(gpu_ctx, lo, hi, p, out)
        serial.append(out)

    ctxs = [capi.Context(0) for _ in pairs]
    outs = [[np.zeros((p.res, p.res, 3), np.uint8) for _ in range(3)] for p in pairs]

    def worker(i):
        for k in range(3):  # eager, capture, replay
            _bake(ctxs[i], views[i][0], views[i][1], pairs[i], outs[i][k])

    with cf.ThreadPoolExecutor(max_workers=len(pairs)) as pool:
        list(pool.map(worker, range(len(pairs))))
    for i in range(len(pairs)):
        for k in range(3):
            assert np.array_equal(outs[i][k], serial[i]), (i, k)
    for c in ctxs:
        c.close()
