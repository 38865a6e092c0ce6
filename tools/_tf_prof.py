import os, sys, json, tempfile, subprocess, threading, time
sys.path.insert(0, os.getcwd())
import torch, bench as B
from torch.profiler import ProfilerActivity, profile
from paper_2605_26137_b200 import capi, fixtures as fx
p = fx.config_pair("B")
stream = torch.cuda.current_stream()
ctx = capi.Context(0, stream.cuda_stream)
lo = capi.DeviceMesh(ctx, p.lowpoly)
samples = []
stop = False
def smi():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_event_reasons.active", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
        samples.append(out); time.sleep(0.05)
th = threading.Thread(target=smi); th.start()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    B.texfuse_bench(ctx, lo, p, 10)
stop = True; th.join()
print("smi:", samples[:3], samples[-3:])
fd, path = tempfile.mkstemp(suffix=".json"); os.close(fd)
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
# group kernels into calls: each call starts with k_valid_bounds
calls = []; cur = None
for e in ev:
    n = e["name"].replace("(anonymous namespace)", "anon").split("(")[0].replace("void ", "").split("::")[-1]
    if n.startswith("k_valid_bounds"):
        cur = {}; calls.append(cur)
    if cur is not None:
        cur[n] = cur.get(n, 0.0) + e["dur"]
for i, c in enumerate(calls):
    print(i, " ".join(f"{k[:12]}={v:.0f}" for k, v in sorted(c.items(), key=lambda kv: -kv[1])[:5]))
