"""Diagnose the host-buffer (e2e) bake path timing."""
import ctypes, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_26137_b200 import capi, fixtures as fx
from paper_2605_26137_b200.mesh import TriangleMesh
pair = fx.config_pair("B")
ctx = capi.Context(0, torch.cuda.current_stream().cuda_stream)
def pinned(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    return t.numpy()
lo, hi = pair.lowpoly, pair.dense
lo_p = TriangleMesh(pinned(lo.positions), pinned(lo.faces), uvs=pinned(lo.uvs), face_uvs=pinned(lo.face_uvs))
hi_p = TriangleMesh(pinned(hi.positions), pinned(hi.faces))
out = torch.empty((pair.res, pair.res, 3), dtype=torch.uint8).pin_memory().numpy()
lv, hv = lo_p.view(), hi_p.view()
st = capi.MfBakeStats()
ctx.set_timing(True)
for i in range(6):
    t0 = time.perf_counter()
    capi.check(ctx.lib.mf_bake_normal_map(ctx.h, ctypes.byref(lv), ctypes.byref(hv), pair.res, pair.bbox_diagonal,
               pair.max_distance_fraction, 4, ctypes.c_void_p(out.ctypes.data), None, None, ctypes.byref(st)))
    t1 = time.perf_counter()
    print(f"wall {1e3*(t1-t0):.2f} ms", {k: round(v, 3) for k, v in st.as_dict().items() if k.startswith('ms')})
d = torch.empty(hi_p.positions.nbytes, dtype=torch.uint8, device="cuda")
src = torch.from_numpy(hi_p.positions.view(np.uint8).reshape(-1))
print("src pinned:", src.is_pinned())
torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(src, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"H2D {hi_p.positions.nbytes/1e6:.1f} MB in {1e3*(t1-t0):.3f} ms")
t0 = time.perf_counter()
for i in range(1000): ctx.lib.mf_abi_version()
print(f"trivial ctypes call {1e3*(time.perf_counter()-t0):.3f} us")
import ctypes as C
t0 = time.perf_counter()
rc = ctx.lib.mf_bake_normal_map(ctx.h, C.byref(lv), C.byref(hv), pair.res, pair.bbox_diagonal, pair.max_distance_fraction, 4, C.c_void_p(out.ctypes.data), None, None, C.byref(st))
t1 = time.perf_counter()
print("direct call", rc, f"{1e3*(t1-t0):.3f} ms")
