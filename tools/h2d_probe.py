"""H2D/D2H copy-engine probe: pinned host <-> device throughput for one copy
vs two concurrent copies on two streams (informs the e2e overlap design)."""
import torch, time
N = 24 * 1024 * 1024
h = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def one(): d.copy_(h, non_blocking=True)
def two():
    ev = torch.cuda.Event(); ev.record()
    with torch.cuda.stream(s1):
        s1.wait_event(ev); d[:N//2].copy_(h[:N//2], non_blocking=True)
    with torch.cuda.stream(s2):
        s2.wait_event(ev); d[N//2:].copy_(h[N//2:], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
ss = [torch.cuda.Stream() for _ in range(4)]
def four():
    ev = torch.cuda.Event(); ev.record()
    q = N // 4
    for k, st in enumerate(ss):
        with torch.cuda.stream(st):
            st.wait_event(ev); d[k * q:(k + 1) * q].copy_(h[k * q:(k + 1) * q], non_blocking=True)
    for st in ss: torch.cuda.current_stream().wait_stream(st)
def down(): h.copy_(d, non_blocking=True)
for name, fn in (("h2d one", one), ("h2d two streams", two), ("h2d four streams", four), ("d2h one", down)):
    ms = t(fn); print(f"{name}: {ms:.3f} ms  {N / ms / 1e6:.1f} GB/s")
