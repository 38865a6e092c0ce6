"""Per-kernel timeline of the fused device bake (graph replays) via CUPTI
(torch.profiler / kineto): start offset from the bake's first kernel, duration
and stream of every kernel, concurrent as they really ran (no serialisation,
unlike ncu). Diagnostic only.

   python tools/timeline.py [config] [bakes] > gpurun_out/timeline.txt
"""
import json
import os
import statistics
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2605_26137_b200 import capi, fixtures as fx

name = sys.argv[1] if len(sys.argv) > 1 else "B"
bakes = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p = fx.config_pair(name)
res = p.res
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)  # the context launches on it (the default stream would be NULL)
ctx = capi.Context(0, stream.cuda_stream)
lo = capi.DeviceMesh(ctx, p.lowpoly)
hi = capi.DeviceMesh(ctx, p.dense)
rgb = torch.empty((res, res, 3), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


E2E = os.environ.get("TL_E2E") == "1"  # the host-buffer entry point (pinned inputs / output) instead
if E2E:
    import numpy as np

    from paper_2605_26137_b200 import meshforge as mf

    def _pin(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    if os.environ.get("TL_PAGEABLE") == "1":  # numpy (pageable) inputs and output
        hlo, hhi, hout = p.lowpoly, p.dense, np.zeros((res, res, 3), np.uint8)
    else:
        hlo = mf.TriangleMesh(_pin(p.lowpoly.positions), _pin(p.lowpoly.faces), uvs=_pin(p.lowpoly.uvs),
                              face_uvs=_pin(p.lowpoly.face_uvs))
        hhi = mf.TriangleMesh(_pin(p.dense.positions), _pin(p.dense.faces))
        hout = torch.empty((res, res, 3), dtype=torch.uint8).pin_memory().numpy()


def bake():
    if E2E:
        mf.bake_normal_map(hlo, hhi, res, p.bbox_diagonal, p.max_distance_fraction, 4, out=hout, ctx=ctx)
        return
    capi.check(ctx.lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, res, p.bbox_diagonal, p.max_distance_fraction, 4,
                                              0, res, rgb.data_ptr(), None))


for _ in range(5):  # eager, capture, replays
    bake()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(bakes):
        flush.zero_()
        torch.cuda.synchronize()
        bake()
        torch.cuda.synchronize()
fd, path = tempfile.mkstemp(suffix=".json")
os.close(fd)
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
os.unlink(path)
ev.sort(key=lambda e: e["ts"])
# split into bakes: the flush kernel (FillFunctor) separates them
groups, cur = [], []
for e in ev:
    if "FillFunctor" in e["name"] or "fill" in e["name"].lower() and "vectorized" in e["name"]:
        if cur:
            groups.append(cur)
        cur = []
        continue
    cur.append(e)
if cur:
    groups.append(cur)


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("mfb::", "")
    if n.startswith("void "):
        n = n[5:]
    if "cub::" in n:
        return n.split("<")[0]
    return n.split("(")[0][:60]


rows = defaultdict(list)
spans = []
for g in groups:
    t0 = g[0]["ts"]
    t1 = max(e["ts"] + e["dur"] for e in g)
    spans.append(t1 - t0)
    seen = defaultdict(int)
    for e in g:
        k = short(e["name"]) if e.get("cat") == "kernel" else e["cat"] + ":" + e["name"][:40]
        seen[k] += 1
        rows[(k, seen[k])].append((e["ts"] - t0, e["dur"], e["args"].get("stream", -1)))
print(f"# config {name}: {len(groups)} bakes, span us: " + ", ".join(f"{s:.1f}" for s in spans))
print(f"# median span {statistics.median(spans):.1f} us; per kernel: median start, end, dur (us), stream")
order = sorted(rows.items(), key=lambda kv: statistics.median(v[0] for v in kv[1]))
for (k, i), v in order:
    st = statistics.median(x[0] for x in v)
    du = statistics.median(x[1] for x in v)
    print(f"{st:8.1f} {st + du:8.1f} {du:7.1f}  s{v[0][2]:<3} {k}{'' if i == 1 else f' #{i}'}")
