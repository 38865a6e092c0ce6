"""Median host-buffer bake time (pinned inputs/outputs) over N calls at config B:
   python tools/e2e_ab.py [N]   (A/B via env switches, e.g. MFB_E2E_BANDS=0)"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_26137_b200 import fixtures as fx
from paper_2605_26137_b200 import meshforge as mf

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
p = fx.config_pair("B")
res = p.res


def pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()


lo = mf.TriangleMesh(pinned(p.lowpoly.positions), pinned(p.lowpoly.faces), uvs=pinned(p.lowpoly.uvs),
                     face_uvs=pinned(p.lowpoly.face_uvs))
hi = mf.TriangleMesh(pinned(p.dense.positions), pinned(p.dense.faces))
out = torch.empty((res, res, 3), dtype=torch.uint8).pin_memory().numpy()
ts = []
for i in range(n + 3):
    t = time.perf_counter()
    mf.bake_normal_map(lo, hi, res, p.bbox_diagonal, p.max_distance_fraction, 4, out=out)
    ts.append((time.perf_counter() - t) * 1e3)
ts = ts[3:]
print(os.environ.get("TAG", ""), "median %.3f ms  min %.3f  mean %.3f" % (statistics.median(ts), min(ts), statistics.mean(ts)))
