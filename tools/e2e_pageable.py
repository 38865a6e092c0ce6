"""Median host-buffer bake time at config B, pinned and pageable (numpy)
inputs/outputs, over N calls (A/B of library variants via MFB_LIB):
   python tools/e2e_pageable.py [N]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_26137_b200 import fixtures as fx
from paper_2605_26137_b200 import meshforge as mf

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
p = fx.config_pair("B")
res = p.res


def pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()


cases = {
    "pinned": (mf.TriangleMesh(pinned(p.lowpoly.positions), pinned(p.lowpoly.faces), uvs=pinned(p.lowpoly.uvs),
                               face_uvs=pinned(p.lowpoly.face_uvs)),
               mf.TriangleMesh(pinned(p.dense.positions), pinned(p.dense.faces)),
               torch.empty((res, res, 3), dtype=torch.uint8).pin_memory().numpy()),
    "pageable": (p.lowpoly, p.dense, np.zeros((res, res, 3), np.uint8)),
}
line = []
for name, (lo, hi, out) in cases.items():
    ts = []
    for i in range(n + 3):
        t = time.perf_counter()
        mf.bake_normal_map(lo, hi, res, p.bbox_diagonal, p.max_distance_fraction, 4, out=out)
        if i >= 3:
            ts.append((time.perf_counter() - t) * 1e3)
    line.append(f"{name} {statistics.median(ts):.3f} ms")
print(os.environ.get("MFB_LIB", "base"), "  ".join(line))
