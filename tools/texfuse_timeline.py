"""Per-kernel CUPTI timeline of one mf_fuse_views_dev call (10 standard views
at 1024^2 onto the config-B 2048^2 G-buffer) after warm-up. Diagnostic."""
import json
import os
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2605_26137_b200 import capi, fixtures as fx  # noqa: E402

p = fx.config_pair("B")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)  # the context launches on it (the default stream would be NULL)
ctx = capi.Context(0, stream.cuda_stream)
lo = capi.DeviceMesh(ctx, p.lowpoly)
print(bench.texfuse_bench(ctx, lo, p, int(os.environ.get("TF_STEPS", "5")))["ms"], "ms (bench timing)")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    bench.texfuse_bench(ctx, lo, p, 3)
fd, path = tempfile.mkstemp(suffix=".json")
os.close(fd)
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
os.unlink(path)
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    k = e["name"].split("(")[0].replace("void ", "").split("::")[-1][:40]
    agg[k][0] += 1
    agg[k][1] += e["dur"]
for k, (n, d) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"{d:10.1f} us {n:6d}x  {k}")
