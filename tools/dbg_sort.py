"""Diagnostic: the LBVH leaf order vs numpy's stable Morton argsort."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2605_26137_b200 import fixtures as fx, meshforge as mf  # noqa: E402
from test_gpu_spatial import _morton30  # noqa: E402

for nlat in [int(a) for a in (sys.argv[1:] or ["64", "100", "160"])]:
    t0 = time.time()
    m = fx.star_blob(3, nlat, nlat)
    _, links, order = mf.Bvh(m).export()
    k = _morton30(m)
    exp = np.argsort(k, kind="stable")
    bad = np.nonzero(order != exp)[0]
    ks = k[order].astype(np.int64)
    print(m.face_count(), "tiles", -(-m.face_count() // 8192), "mismatch", len(bad),
          "sorted", bool((np.diff(ks) >= 0).all()), "perm", bool(np.array_equal(np.sort(order), np.arange(m.face_count()))),
          "first bad", bad[:4], "keys", k[order[bad[:4]]], k[exp[bad[:4]]], f"{time.time() - t0:.1f}s", flush=True)
