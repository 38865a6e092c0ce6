"""Host wall time vs GPU span of the pinned host-buffer bake (mf_bake_normal_map),
per call: where an end-to-end call spends time outside the GPU's work.

   MFB_TRACE=1 MFB_TRACE_MARKS=1 python tools/e2e_probe.py [config] [calls]
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2605_26137_b200 import capi, fixtures as fx

name = sys.argv[1] if len(sys.argv) > 1 else "A"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 10
p = fx.config_pair(name)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = capi.Context(0, stream.cuda_stream)
lo_p, hi_p, _ = bench._pinned_pair(p)
out = torch.empty((p.res, p.res, 3), dtype=torch.uint8).pin_memory().numpy()
lv, hv = lo_p.view(), hi_p.view()
st = capi.MfBakeStats()
for timing in (0, 1):
    ctx.set_timing(bool(timing))
    for k in range(calls):
        t = time.perf_counter()
        capi.check(ctx.lib.mf_bake_normal_map(ctx.h, ctypes.byref(lv), ctypes.byref(hv), p.res, p.bbox_diagonal,
                                              p.max_distance_fraction, 4, ctypes.c_void_p(out.ctypes.data), None,
                                              None, ctypes.byref(st)))
        wall = (time.perf_counter() - t) * 1e3
        print(f"timing={timing} call {k}: host wall {wall:.3f} ms" +
              (f", GPU t0->t3 {st.ms_total:.3f} ms, upload {st.ms_upload:.3f}, download {st.ms_download:.3f}"
               if timing else ""), flush=True)
