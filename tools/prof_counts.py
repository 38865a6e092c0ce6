"""Traversal counters (MFB_PROF=1) of one config bake: internal node visits,
leaves and triangle tests per query, printed by the library on stderr."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_26137_b200 import capi, fixtures as fx
import ctypes
name = sys.argv[1] if len(sys.argv) > 1 else "B"
pair = fx.config_pair(name)
ctx = capi.Context(0)
lo, hi = capi.DeviceMesh(ctx, pair.lowpoly), capi.DeviceMesh(ctx, pair.dense)
import torch
rgb = torch.empty((pair.res, pair.res, 3), dtype=torch.uint8, device="cuda")
ctx.set_timing(True)  # eager (the counters are printed per eager launch)
capi.check(ctx.lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, pair.res, pair.bbox_diagonal,
                                          pair.max_distance_fraction, 4, 0, pair.res, rgb.data_ptr(), None))
ctx.synchronize()
