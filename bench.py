#!/usr/bin/env python
"""Benchmark: baked texels/s (+ BVH rays/s) of the fused B200 normal bake.

Workloads (BASELINE.json configs, synthetic Appendix-B pairs):
  N = 1 (default): config B - dense G(224) = 1,003,520 faces -> lowpoly G(32)
        = 20,480 faces, 20-chart atlas, 2048^2, maxDistanceFraction 0.01,
        dilation radius 4, one asset on one B200.
  N > 1 (default): config C - the same meshes at 4096^2, ONE atlas row-sharded
        across the N GPUs (valid-balanced row slabs + dilation halo, the BVH
        replicated per rank), gathered by the producing dilation kernel's
        stores into every rank's atlas over CUDA IPC peer memory (NVLink /
        NVSwitch; `--gather nccl` = NCCL all-gather + assembly) -> "scaling":
        "strong"; plus config D as 8 independent assets per GPU (the 64-asset
        batch at N = 8, no collective), reported under "batch_d".
One step = one whole bake: dense vertex normals + LBVH build + lowpoly wedge
frames/reliability + raster + closest-point transfer + dilation, i.e.
dilateSeams(transferNormals(rasterizeGBuffer(lo), hi, diag), g, 4) of the
reference (test_bake.cpp:205-206), with the meshes already resident in HBM.

`value`  = N_v / t_step   (baked texels/s, device time, CUDA events, max over ranks)
`e2e`    = the same bake through the host-buffer C ABI (N = 1: mf_bake_normal_map
           from pinned host memory; N > 1: per rank, mesh upload + validation,
           the sharded bake and its gather, D2H of the atlas), copies inside
           the timed region.
`--gpus N` without torchrun re-launches itself under torch.distributed.run
(one rank per GPU, 127.0.0.1 rendezvous).

`--impl reference` times the reference's own CPU implementation (the
reference TUs compiled in place, oracle/_ref/libmfref.so; the C restatement
oracle/build/liboracle.so if that is absent) on the host cores, rank 0 only,
on the same workload and config dict as `--impl ours`.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "baked texels/sec (2048^2 atlas, 1M-face dense source, config B)"
METRICS = {
    "A": "baked texels/sec (512^2 atlas, 200k-face dense source, config A)",
    "B": METRIC,
    "C": "baked texels/sec (4096^2 atlas, 1M-face dense source, config C)",
    "D": "baked texels/sec (1024^2 atlas, 500k-face dense source, config D asset)",
    "E": "baked texels/sec (4096^2 atlas, 4M-face dense source, large cage offset, config E)",
}
UNIT = "texels/s"
CONSTANTS = os.path.join(ROOT, "bench_data", "reference_counters.json")
TRAFFIC = os.path.join(ROOT, "profiles", "k_transfer_ncu.json")  # one `ncu --set full` capture
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
PEAKS_LIB = os.path.join(ROOT, "build", "libmfpeaks.so")  # tools/peaks.cu
N_RAYS = 1_000_000  # SURVEY §8(d) secondary metric: raycastFirst on 10^6 random rays
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
L2_FLUSH = "flushed between timed steps (256 MiB write, outside the per-step events)"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=None, help="A..E (default: B at N = 1, C at N > 1)")
    ap.add_argument("--mode", choices=["auto", "single", "shard", "replicas", "batch"], default="auto",
                    help="auto: single at N = 1, shard at N > 1; replicas: one asset per rank (seed 7 + rank); "
                         "batch: --assets independent assets per GPU")
    ap.add_argument("--shard", action="store_true", help="same as --mode shard")
    ap.add_argument("--gather", choices=["nccl", "peer"], default="peer",
                    help="shard: atlas gather by the dilation kernel storing its rows into every rank's atlas "
                         "over CUDA IPC peer memory (mf_bake_normal_map_dev_publish), or NCCL all-gather")
    ap.add_argument("--assets", type=int, default=8, help="batch: independent assets per GPU (config D: 8)")
    ap.add_argument("--no-batch", action="store_true", help="N > 1: skip the config-D batch line")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rays", action="store_true", help="skip the secondary BVH rays/s metrics")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--launch-selftest", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args(argv)


def resolve(args, world):
    """(mode, config) of this run."""
    mode = "shard" if args.shard else args.mode
    if mode == "auto":
        mode = "shard" if world > 1 else "single"
    if mode == "shard" and world == 1:
        mode = "single"
    name = args.config or {"shard": "C", "batch": "D"}.get(mode, "B")
    return mode, name


def config_dict(name, pair, mode, world, assets=1, seed=None):
    """The workload description both arms print (identical dicts)."""
    par = {"single": "single asset, one GPU",
           "shard": f"rows x{world}: one atlas in valid-balanced row slabs, BVH replicated, atlas gathered",
           "replicas": f"assets x{world}: one asset per GPU, no collective",
           "batch": f"assets x{assets * world}: {assets} per GPU, no collective"}[mode]
    batch = {"shard": 1, "replicas": world, "batch": assets * world}.get(mode, 1)
    return {"workload": workload_desc(name, pair), "global_batch": batch, "seq_len": None, "parallelism": par,
            "l2": L2_FLUSH, "seed": seed}


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(argv, n):
    """`bench.py --gpus N` outside torchrun: re-run under torch.distributed.run
    with one rank per GPU (NCCL init lines on, so the rank count is visible)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + argv
    return subprocess.run(cmd, env=env).returncode


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), int(
        os.environ.get("WORLD_SIZE", "1"))


def workload_desc(name, pair):
    return (f"config {name}: dense G(n) {pair.dense.face_count():,} faces / {pair.dense.vertex_count():,} verts"
            f" -> lowpoly {pair.lowpoly.face_count():,} faces, 20-chart atlas, {pair.res}^2, "
            f"maxDistFrac {pair.max_distance_fraction}, dilation r=4")


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region with NVML
    (every 2 ms; nvidia-smi's 100 ms floor would miss a ~20 ms region),
    falling back to `nvidia-smi -lms 100`."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.stop = threading.Event()
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:  # no NVML: nvidia-smi
            self.nvml = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read, daemon=True)
                self.t.start()
            except OSError:
                self.proc = None
        return self

    def _poll(self):
        n = self.nvml
        while not self.stop.is_set():
            try:
                sm = n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM)
                try:
                    rs = n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    rs = n.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((float(sm), float(self.max_mhz), int(rs)))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        elif getattr(self, "t", None):
            self.t.join(timeout=1)

    def summary(self):
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap"}
        reasons = set()
        sm, mx = [], None
        for v, m, rs in self.samples:
            sm.append(v)
            mx = m
            for bit, nm in names.items():
                if rs & bit:
                    reasons.add(nm)
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"],
                               parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def live_peaks(device):
    """L2 read bandwidth and FP64 FMA throughput measured live on this box
    (tools/peaks.cu; MEASURED_PEAKS.json has only HBM and bf16)."""
    import ctypes
    try:
        lib = ctypes.CDLL(PEAKS_LIB)
    except OSError as e:
        return {"error": f"{PEAKS_LIB}: {e}"}
    lib.mfp_l2_read_gbs.argtypes = [ctypes.c_int, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    lib.mfp_fp64_tflops.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    out = {"source": "live, tools/peaks.cu: 64 MiB L2-resident buffer streamed with ld.global.cg by 4 CTAs/SM "
                     "(best of 5); 8 independent DFMA chains per thread, 8 CTAs/SM (best of 5)"}
    v = ctypes.c_double()
    if lib.mfp_l2_read_gbs(device, 64 << 20, 20, ctypes.byref(v)) == 0:
        out["l2_read_gbs"] = round(v.value, 1)
    if lib.mfp_fp64_tflops(device, ctypes.byref(v)) == 0:
        out["fp64_tflops"] = round(v.value, 2)
    return out


def stage_rooflines(pair, stage, n_queries, counters, hbm, peaks, n_valid=None):
    """SURVEY §8(d) per-stage roofline fractions: streaming stages against HBM,
    the traversal against the measured L2 read bandwidth and the FP64 pipe.
    Times are the eager per-stage CUDA-event times (all kernels of the stage)."""
    res = pair.res
    f, v = pair.dense.face_count(), pair.dense.vertex_count()

    def row(bytes_, ms, peak, unit="GB/s", scale=1e9, note=""):
        if not ms or not peak:
            return None
        a = bytes_ / (ms * 1e-3) / scale
        r = {"algorithmic": bytes_, "ms": round(ms, 4), "achieved": round(a, 1), "peak": peak, "unit": unit,
             "frac": round(a / peak, 4)}
        if note:
            r["note"] = note
        return r

    out = {
        "raster": row(50 * res * res, stage["ms_raster"], hbm,
                      note="50 B x res^2 (G-buffer as the API output); fused path writes only query records"),
        "lbvh": row(148 * f + 24 * v, stage["ms_bvh"], hbm,
                    note="148 F + 24 V; stage also builds the dense vertex normals, side stream, overlapped"),
        # the fused bake resolves the dilation before the transfer: its time is
        # the dilation-links kernel (the copies ride on the transfer epilogue)
        "dilate": row(7 * res * res, stage["ms_dilate"], hbm,
                      note="7 B x res^2 over the dilation-links kernel's time (fused bake: the source choice; "
                           "the copies are stored by the transfer epilogue)"),
    }
    if counters:
        out["transfer_l2"] = row(counters["bytes_per_query"] * n_queries, stage["ms_transfer"],
                                 peaks.get("l2_read_gbs"),
                                 note="W_q x N_q visit bytes against the measured L2 read bandwidth")
        flops = (22 * counters["n_node"] + 80 * counters["n_tri"]) * n_queries
        out["transfer_fp64"] = row(flops, stage["ms_transfer"], peaks.get("fp64_tflops"), unit="TFLOP/s",
                                   scale=1e12, note="(22 N_node + 80 N_tri) x N_q")
    return out


def bvh_rays(ctx, hi, pair, steps):
    """Secondary metrics: Bvh::raycastFirst over 10^6 random rays
    (origins uniform in the dense mesh's box, directions uniform on the sphere)
    and closestPointWithin over 10^6 random points at the bake's search radius,
    both against the dense LBVH, device-resident inputs, CUDA events."""
    import ctypes
    import torch

    from paper_2605_26137_b200 import capi
    lib = ctx.lib
    h = ctypes.c_void_p()
    capi.check(lib.mf_bvh_build(ctx.h, hi.h, ctypes.byref(h)))
    g = torch.Generator(device="cuda").manual_seed(11)
    lo_b = torch.tensor(pair.dense.positions.min(0), device="cuda")
    hi_b = torch.tensor(pair.dense.positions.max(0), device="cuda")
    o = lo_b + (hi_b - lo_b) * torch.rand((N_RAYS, 3), generator=g, device="cuda", dtype=torch.float64)
    d = torch.randn((N_RAYS, 3), generator=g, device="cuda", dtype=torch.float64)
    d /= d.norm(dim=1, keepdim=True)
    face = torch.empty(N_RAYS, dtype=torch.int32, device="cuda")
    t, u, w = (torch.empty(N_RAYS, dtype=torch.float64, device="cuda") for _ in range(3))
    pt = torch.empty((N_RAYS, 3), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(3, min(steps, 10))):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    ms_ray = timed(lambda: capi.check(lib.mf_bvh_raycast_first_dev(
        h, o.data_ptr(), d.data_ptr(), N_RAYS, 0.0, float("inf"), face.data_ptr(), t.data_ptr(), u.data_ptr(),
        w.data_ptr())))
    ray_hits = int((face >= 0).sum())
    max_d = pair.max_distance_fraction * pair.bbox_diagonal
    ms_cp = timed(lambda: capi.check(lib.mf_bvh_closest_within_dev(
        h, o.data_ptr(), N_RAYS, max_d, face.data_ptr(), t.data_ptr(), pt.data_ptr(), None)))
    cp_hits = int((face >= 0).sum())
    # markSurfaceBand's voxel sweep: 256^3 voxel-centre
    # queries at the sign field's truncation radius, device outputs
    band_res = 256
    nb = band_res ** 3
    labels = torch.empty(nb, dtype=torch.uint8, device="cuda")
    bdist = torch.empty(nb, dtype=torch.float32, device="cuda")
    ms_band = timed(lambda: capi.check(lib.mf_surface_band_dev(
        h, band_res, 1.0, 2, None, labels.data_ptr(), bdist.data_ptr(), None)))
    band_voxels = int(labels.sum())
    lib.mf_bvh_destroy(h)
    # castVisibility at the paper's setting (PAPER "BVH ... 512
    # viewpoints"): 512 fibonacci ortho views x 1024^2 pixel rays against the
    # dense mesh, whole host call (upload, centring, LBVH, rays, hit counts)
    vis_views, vis_res = 512, 1024
    hits = np.zeros(pair.dense.face_count(), np.int64)
    mv = pair.dense.view()
    ms_vis = timed(lambda: capi.check(lib.mf_cast_visibility(ctx.h, ctypes.byref(mv), vis_views, vis_res,
                                                             hits.ctypes.data_as(ctypes.c_void_p), None)))
    vis_rays = vis_views * vis_res * vis_res
    # the reference's castVisibility on the host cores, 32 of the views (its
    # views are independent, parallelChunks over views)
    vis_cpu = None
    try:
        lib_ref, kind = _reference_lib()
        t0 = time.perf_counter()
        ref_hits = lib_ref.cast_visibility(pair.dense, 32, vis_res)
        dt = time.perf_counter() - t0
        vis_cpu = {"pixels_per_s": 32 * vis_res * vis_res / dt, "s": round(dt, 3), "views": 32, "kind": kind,
                   "cores": cores()}
        del ref_hits
    except Exception as e:  # noqa: BLE001 - the CPU leg is informative only
        vis_cpu = {"unavailable": str(e)[:120]}
    return {"visibility_pixels_per_s": vis_rays / (ms_vis * 1e-3), "visibility_ms": round(ms_vis, 3),
            "visibility_views": vis_views, "visibility_res": vis_res,
            "visibility_visible_faces": int((hits > 0).sum()),
            "visibility_method": "device z-buffer rasteriser (the reference's face loop, atomicMax keys); "
                                 "whole host call incl. upload and centring",
            "visibility_cpu_reference": vis_cpu,
            "surface_band_voxels_per_s": nb / (ms_band * 1e-3), "surface_band_ms": round(ms_band, 4),
            "surface_band_res": band_res, "surface_band_marked": band_voxels,
            "raycast_rays_per_s": N_RAYS / (ms_ray * 1e-3), "raycast_ms": round(ms_ray, 4), "raycast_hits": ray_hits,
            "closest_within_per_s": N_RAYS / (ms_cp * 1e-3), "closest_within_ms": round(ms_cp, 4),
            "closest_within_hits": cp_hits, "n": N_RAYS,
            "inputs": "uniform origins in the dense bbox, uniform unit directions (seed 11); "
                      "closest-point radius = maxDistFrac x diag"}


def texfuse_bench(ctx, lo, pair, steps, once=False):
    """fuseViews up to the blend (fuse.cpp:292-318) on the
    device over the config-B lowpoly's 2048^2 G-buffer (mf_raster_gbuffer_dev,
    resident in HBM) and the 10 standard views at 1024^2 of the dense mesh
    (mf_render_views), 3-channel synthetic colours: one mf_fuse_views_dev call
    = per view edge mask + 6-level mip chain + backprojection + incidence, then
    the blend. The reference's own fuse.cpp runs one of the views on the host
    cores beside it (its backprojectView / incidenceMap are single-threaded)."""
    import ctypes

    import torch

    from paper_2605_26137_b200 import capi
    from paper_2605_26137_b200 import texfuse as tf
    lib = ctx.lib
    res, vres, k = pair.res, 1024, 10
    n = res * res
    gp, gn, gt, gb = (torch.empty((n, 3), dtype=torch.float32, device="cuda") for _ in range(4))
    gv, gr = (torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(2))
    capi.check(lib.mf_raster_gbuffer_dev(ctx.h, lo.h, res, gp.data_ptr(), gn.data_ptr(), gt.data_ptr(),
                                         gb.data_ptr(), gv.data_ptr(), gr.data_ptr()))
    cams = tf.standard_cameras(0.8)
    face = np.zeros((k, vres, vres), np.int32)
    depth = np.zeros((k, vres, vres), np.float32)
    pos = np.zeros((k, vres, vres, 3), np.float32)
    mv = pair.dense.view()
    capi.check(lib.mf_render_views(ctx.h, ctypes.byref(mv), cams.ctypes.data_as(ctypes.c_void_p), k, vres, None, 0,
                                   face.ctypes.data_as(ctypes.c_void_p), depth.ctypes.data_as(ctypes.c_void_p),
                                   pos.ctypes.data_as(ctypes.c_void_p), None))
    fg = (face >= 0)[..., None]
    col = ((0.5 + 0.5 * np.sin(np.concatenate([7.0 * pos[..., :1], 5.0 * pos[..., 1:2] + 1.0,
                                                3.0 * pos[..., 2:3]], -1))) * fg).astype(np.float32)
    dface, ddepth, dpos, dcol = (torch.from_numpy(a).cuda() for a in (face, depth, pos, col))
    out = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    filled = torch.empty(n, dtype=torch.uint8, device="cuda")
    priors = np.array(tf.standard_view_priors())
    diag = pair.bbox_diagonal

    def call():
        capi.check(lib.mf_fuse_views_dev(ctx.h, res, gp.data_ptr(), gn.data_ptr(), gv.data_ptr(), k,
                                          cams.ctypes.data_as(ctypes.c_void_p), vres, dpos.data_ptr(),
                                          dface.data_ptr(), ddepth.data_ptr(), 3, dcol.data_ptr(),
                                          priors.ctypes.data_as(ctypes.c_void_p), diag, None, out.data_ptr(),
                                          filled.data_ptr()))
    call()
    torch.cuda.synchronize()
    if once:  # (profiling: one call)
        return None
    stream = torch.cuda.current_stream()
    ts = []
    for _ in range(max(3, min(steps, 10))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        call()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    if os.environ.get("MFB_TF_TRACE"):
        print("texfuse call ms:", " ".join(f"{t:.3f}" for t in ts), file=sys.stderr)
    ms = statistics.median(ts)
    n_valid = int(gv.sum())
    n_filled = int(filled.sum())
    line = {"ms": round(ms, 3), "views": k, "view_res": vres, "atlas_res": res, "valid_texels": n_valid,
            "filled_texels": n_filled, "texel_views_per_s": n_valid * k / (ms * 1e-3),
            "call": "mf_fuse_views_dev: every image resident in HBM (G-buffer from mf_raster_gbuffer_dev)"}
    # the reference's fuse.cpp on the host cores: edgeMask + buildMips +
    # backprojectView + incidenceMap of view 0 (single-threaded as shipped)
    try:
        from oracle import bindings
        if bindings.ref_available():
            r = bindings.ref()
            gpos, gnrm, gval = gp.cpu().numpy(), gn.cpu().numpy(), gv.cpu().numpy()
            t0 = time.perf_counter()
            m = r.edge_mask(pos[0], face[0], diag, 0.02)
            chain, nm = r.build_mips(col[0], 6, 0.2)
            r.backproject_view(gpos, gval, res, cams[0], vres, 3, nm, chain, m)
            r.incidence_map(gpos, gnrm, gval, res, cams[0], vres, depth[0], diag, 0.005)
            dt = time.perf_counter() - t0
            line["cpu_reference"] = {"s_per_view": round(dt, 3), "texel_views_per_s": n_valid / dt, "cores": 1,
                                     "kind": "reference", "sample": "view 0 of 10 (edgeMask, buildMips, "
                                     "backprojectView, incidenceMap; the blend excluded)"}
    except Exception as e:  # noqa: BLE001 - informative only
        line["cpu_reference"] = {"unavailable": str(e)[:120]}
    return line


def transfer_traffic():
    """dram__bytes_read + dram__bytes_write of the transfer kernel from the
    committed `ncu --set full` capture summary (profiles/k_transfer_ncu.json),
    with that launch's whole record."""
    try:
        with open(TRAFFIC) as f:
            d = json.load(f)
        launch = next(x for x in d["launches"] if "k_transfer" in x["kernel"])
        return float(launch["dram_bytes"]), d.get("source"), launch
    except (OSError, KeyError, StopIteration, ValueError):
        return None, None, None


def transfer_algorithmic_bytes(name, n_queries, n_valid, res):
    """transfer bytes per query W_q = 50 (G-buffer read) + 3 (RGB8
    write) + 64*N_node + 84*N_tri + 72 (winner's vertex normals), N_node/N_tri =
    the reference best-first traversal's mean nodes popped / triangles tested
    per query, measured once with the instrumented reference harness on this
    exact input (bench_data/reference_counters.json)."""
    try:
        with open(CONSTANTS) as f:
            c = json.load(f)[name]
        n_node, n_tri = float(c["n_node"]), float(c["n_tri"])
    except (OSError, KeyError):
        return None, None
    per_q = 50 + 3 + 64 * n_node + 84 * n_tri + 72
    return per_q * n_queries, dict(n_node=n_node, n_tri=n_tri, bytes_per_query=per_q)


# ----------------------------------------------------------------------------- ours
class Dist:
    """torch.distributed plumbing of one bench rank: NCCL when every rank has
    its own GPU, gloo when ranks share one (a single-GPU test of the N > 1
    path); small host-side reductions either way."""

    def __init__(self):
        import torch
        self.rank, self.local_rank, self.world = dist_env()
        self.on = "RANK" in os.environ
        ndev = torch.cuda.device_count()
        self.device = self.local_rank % max(ndev, 1)
        self.shared_gpu = self.on and ndev < self.world
        torch.cuda.set_device(self.device)
        self.backend = None
        if self.on:
            import torch.distributed as dist
            self.backend = "gloo" if self.shared_gpu else "nccl"
            if self.backend == "nccl":
                os.environ.setdefault("NCCL_DEBUG", "INFO")
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))
            else:
                dist.init_process_group("gloo")

    def _reduce(self, vals, op):
        if not self.on:
            return list(vals)
        import torch
        import torch.distributed as dist
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor(list(vals), dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=op)
        return t.tolist()

    def max(self, *vals):
        import torch.distributed as dist
        return self._reduce(vals, dist.ReduceOp.MAX if self.on else None)

    def min(self, *vals):
        import torch.distributed as dist
        return self._reduce(vals, dist.ReduceOp.MIN if self.on else None)

    def sum(self, *vals):
        import torch.distributed as dist
        return self._reduce(vals, dist.ReduceOp.SUM if self.on else None)

    def barrier(self):
        if self.on:
            import torch.distributed as dist
            if self.backend == "nccl":
                dist.barrier(device_ids=[self.device])
            else:
                dist.barrier()

    def close(self):
        if self.on:
            import torch.distributed as dist
            dist.destroy_process_group()


def timed_steps(d, step, steps, warmup, stream, flush, clk_device):
    """W untimed warm-up steps, then K timed steps bracketed by a barrier and a
    device synchronize on both sides; per-step CUDA events on the launching
    stream with the L2 flushed (untimed) in between. Returns (mean ms over
    the K steps, clock summary)."""
    import torch
    for _ in range(max(warmup, 3)):
        step()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    d.barrier()
    torch.cuda.synchronize()
    with ClockSampler(clk_device) as clk:
        for i in range(steps):
            flush.zero_()
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    d.barrier()
    return sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / steps, clk.summary()


def run_ours(args, argv_mode, name):
    import ctypes

    import torch

    d = Dist()
    rank, world = d.rank, d.world
    mode = argv_mode
    from paper_2605_26137_b200 import capi, fixtures as fx
    from paper_2605_26137_b200 import meshforge as mf

    if mode == "batch":
        line = run_batch(args, d, name)
        d.close()
        return line

    seed = fx.CONFIGS[name]["seed"] + (rank if mode == "replicas" else 0)
    pair = fx.config_pair(name, seed=seed)
    res = pair.res
    # one non-default stream for everything timed here: the context launches
    # on it, and the L2 flush, the CUDA events and torch's own work are issued
    # on it too (torch's default stream would be handed to the library as
    # NULL, and the context would then launch on a stream of its own that
    # the events do not bracket)
    stream = torch.cuda.Stream(device=d.device)
    torch.cuda.set_stream(stream)
    ctx = capi.Context(d.device, stream.cuda_stream)
    lib = ctx.lib
    lo = capi.DeviceMesh(ctx, pair.lowpoly)
    hi = capi.DeviceMesh(ctx, pair.dense)
    diag = pair.bbox_diagonal
    frac = pair.max_distance_fraction
    rgb = torch.empty((res, res, 3), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    st = capi.MfBakeStats()

    row_b, row_e = 0, res
    shard_ranges = None
    peer = None
    gather = None
    if mode == "shard":
        # one atlas, rows balanced by valid texels, gathered on every rank
        from paper_2605_26137_b200 import sharding
        counts = np.zeros(res, np.int64)
        capi.check(lib.mf_coverage_rows(ctx.h, lo.h, res, ctypes.c_void_p(counts.ctypes.data)))
        shard_ranges = sharding.balanced_row_ranges(counts, world)
        row_b, row_e = shard_ranges[rank]
        rows_max = max(e - b for b, e in shard_ranges)
        slab = torch.empty((rows_max, res, 3), dtype=torch.uint8, device="cuda")
        gather = args.gather
        if gather == "peer":
            ok = 1.0
            try:
                peer = sharding.PeerAtlas(ctx, res)
            except Exception as e:  # noqa: BLE001 - fall back to NCCL for every rank
                print(f"[bench rank {rank}] peer-memory atlas unavailable ({e}); NCCL all-gather", file=sys.stderr)
                ok = 0.0
            if d.min(ok)[0] < 1.0:
                if peer is not None:
                    peer.close()
                peer = None
                gather = "nccl"
        if gather == "nccl":
            gathered = [torch.empty_like(slab) for _ in range(world)]

    def step(stats=None):
        if shard_ranges is None:
            capi.check(lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, res, diag, frac, 4, 0, res,
                                                  rgb.data_ptr(), stats))
            return
        if peer is not None:  # rows stored into every rank's atlas by the dilation kernel
            capi.check(lib.mf_bake_normal_map_dev_publish(ctx.h, lo.h, hi.h, res, diag, frac, 4, row_b, row_e,
                                                          peer.dst, peer.n, stats))
            d.barrier()
            return
        capi.check(lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, res, diag, frac, 4, row_b, row_e,
                                              slab.data_ptr(), stats))
        if d.backend == "nccl":
            torch.distributed.all_gather(gathered, slab)
            rgb.copy_(sharding.assemble(gathered, shard_ranges))
        else:  # ranks sharing one GPU (test mode): gather through the host
            host = [torch.empty_like(slab, device="cpu") for _ in range(world)]
            torch.distributed.all_gather(host, slab.cpu())
            rgb.copy_(sharding.assemble(host, shard_ranges).to("cuda"))

    ms_step, clocks = timed_steps(d, lambda: step(st), args.steps, args.warmup, stream, flush, d.device)
    n_valid, n_queries, hits = st.valid_texels, st.queries, st.hits
    # graph replays bypass the host launch counter: count one eager bake's
    launches = launches_per_bake(ctx, step) * args.steps
    # stage breakdown + the transfer kernel's own duration: the same bake run
    # eagerly with CUDA events around each stage on the launching stream
    ctx.set_timing(True)
    stage = {k: [] for k in ("ms_prepare", "ms_bvh", "ms_raster", "ms_transfer", "ms_dilate", "ms_total")}
    for _ in range(max(3, min(args.steps, 10))):
        flush.zero_()
        step(st)
        dd = st.as_dict()
        for k in stage:
            stage[k].append(dd[k])
    ctx.set_timing(False)
    ms_transfer = statistics.mean(stage["ms_transfer"])

    # aggregate over ranks: max time, summed work (slabs overlap by the
    # dilation halo: a sharded atlas counts each texel once)
    t_max, t_xfer_max = d.max(ms_step, ms_transfer)
    agg_nv, agg_nq = d.sum(n_valid, n_queries)
    extra = {}
    if shard_ranges is not None:
        agg_nv, agg_nq = float(_n_valid(pair)), float(n_queries_full(name, pair))
        extra["shards"] = {"ranges": shard_ranges, "gather": gather,
                           "gather_method": ("dilation kernel stores into every rank's atlas over CUDA IPC "
                                             "peer memory" if gather == "peer" else
                                             ("NCCL all-gather + assembly" if d.backend == "nccl"
                                              else "gloo host all-gather (ranks share one GPU: test mode)")),
                           "backend": d.backend, "shared_gpu": d.shared_gpu}
        # the gathered atlas equals a single-GPU bake of the whole atlas
        full = torch.empty((res, res, 3), dtype=torch.uint8, device="cuda")
        capi.check(lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, res, diag, frac, 4, 0, res, full.data_ptr(),
                                              None))
        torch.cuda.synchronize()
        atlas = peer.atlas if peer is not None else rgb
        eq = float(torch.equal(atlas, full))
        extra["shards"]["gather_check"] = bool(d.max(1.0 - eq)[0] == 0.0)
        # the same config on one GPU (rank 0), for the strong-scaling comparison
        if rank == 0:
            one = lambda: capi.check(lib.mf_bake_normal_map_dev(  # noqa: E731
                ctx.h, lo.h, hi.h, res, diag, frac, 4, 0, res, full.data_ptr(), None))
            for _ in range(3):
                one()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
            for i in range(args.steps):
                flush.zero_()
                ev[2 * i].record(stream)
                one()
                ev[2 * i + 1].record(stream)
            torch.cuda.synchronize()
            ms1 = sum(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(args.steps)) / args.steps
            extra["single_gpu_same_config"] = {"ms_per_step": ms1, "value": agg_nv / (ms1 * 1e-3), "unit": UNIT,
                                               "note": "whole atlas on rank 0's GPU alone, same timing rules"}
        del full

    # secondary BVH metrics and the live L2 / FP64 peaks (rank 0, N = 1 only:
    # they are single-GPU numbers)
    rays = bvh_rays(ctx, hi, pair, args.steps) if rank == 0 and world == 1 and not args.no_rays else None
    texfuse = texfuse_bench(ctx, lo, pair, args.steps) if rank == 0 and world == 1 and not args.no_rays else None
    peaks = live_peaks(d.device) if rank == 0 else {}

    # end-to-end through the public host-buffer API
    e2e = None
    if not args.no_e2e:
        if shard_ranges is not None:
            e2e = run_e2e_shard(args, d, ctx, pair, shard_ranges, peer, gather)
        else:
            e2e = run_e2e(args, d, ctx, pair)

    batch_d = None
    if world > 1 and mode == "shard" and not args.no_batch:
        batch_d = run_batch(args, d, "D", assets=8, as_line=False)

    if rank != 0:
        d.close()
        return None

    peak, peak_src = hbm_peak()
    alg_bytes, counters = transfer_algorithmic_bytes(name, n_queries, n_valid, res)
    stage_mean = {k: statistics.mean(v) for k, v in stage.items()}
    stages_rl = stage_rooflines(pair, stage_mean, n_queries, counters, peak, peaks, n_valid)
    roofline = None
    if alg_bytes is not None:
        # the traversal's node/triangle bytes are served from L2
        # (its DRAM traffic, `traffic`, is ~5% of them), so its roofline is the
        # measured L2 read bandwidth. The §8(d) bytes are node/triangle VISITS
        # (the reference's best-first loop's), not DRAM or L2 transactions;
        # `l2_actual` is the kernel's measured L2 traffic from the committed
        # ncu capture of the same kernel.
        achieved = alg_bytes / (ms_transfer * 1e-3) / 1e9
        traffic, traffic_src, ncu = transfer_traffic()
        l2 = peaks.get("l2_read_gbs")
        roofline = {"bound": "l2" if l2 else "hbm", "kernel": "k_transfer_t (closest-point traversal + encode)",
                    "achieved": round(achieved, 1), "peak": l2 or peak, "unit": "GB/s",
                    "frac": round(achieved / (l2 or peak), 4), "traffic": traffic, "traffic_source": traffic_src,
                    "peak_source": ("measured live: L2 read bandwidth, tools/peaks.cu" if l2 else peak_src),
                    "hbm_peak": peak, "hbm_peak_source": peak_src,
                    "bytes_model": "SURVEY 8(d) visit bytes W_q x N_q (node/triangle visits of the reference's "
                                   "best-first loop), served from L1/L2",
                    "algorithmic_bytes_per_launch": alg_bytes, "ms_per_launch": round(ms_transfer, 4),
                    "per_query": counters}
        if ncu and l2:
            l2b = ncu.get("l2_sectors", 0) * 32.0
            dur = ncu.get("duration_ns")
            if l2b and dur:
                roofline["l2_actual"] = {
                    "bytes_per_launch": l2b, "gbs": round(l2b / dur, 1), "frac": round(l2b / dur / l2, 4),
                    "issue_active_pct": ncu.get("issue_active_pct"),
                    "threads_per_instruction": ncu.get("threads_per_instruction"),
                    "source": traffic_src}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(pair, name, ctx=ctx, gpu_rgb=rgb.cpu().numpy())
    line = {
        "metric": METRICS.get(name, METRIC), "value": agg_nv / (t_max * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t_max,
        "higher_is_better": True, "scaling": "strong" if shard_ranges else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (deterministic geodesic blob pair, Appendix B of SURVEY.md)",
        "config": config_dict(name, pair, mode, world, seed=seed if mode != "replicas" else fx.CONFIGS[name]["seed"]),
        "rays_per_s": agg_nq / (t_xfer_max * 1e-3),
        "n_valid_texels": n_valid, "n_queries": n_queries, "hits": hits,
        "stage_ms": {k: round(statistics.mean(v), 4) for k, v in stage.items()},
        "roofline": roofline, "stage_rooflines": stages_rl, "peaks": peaks, "bvh": rays, "texfuse": texfuse,
        "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks,
    }
    line.update(extra)
    if batch_d is not None:
        line["batch_d"] = batch_d
    d.close()
    return line


def run_batch(args, d, name, assets=None, as_line=True):
    """K independent assets per GPU, each on its own
    context (own stream + side streams, own captured graph), driven by K host
    threads (ctypes drops the GIL in the call). One step = all K bakes;
    value = sum of valid texels over all assets of all ranks / max-rank time.
    Device time: one event on the launch stream that every asset stream waits
    on, and one after the launch stream joins every asset stream."""
    import concurrent.futures as cf

    import torch

    from paper_2605_26137_b200 import capi, fixtures as fx

    k = assets or args.assets
    rank, world = d.rank, d.world
    base = fx.CONFIGS[name]["seed"] + rank * k
    pairs = [fx.config_pair(name, seed=base + i) for i in range(k)]
    streams = [torch.cuda.Stream() for _ in range(k)]
    ctxs = [capi.Context(d.device, s.cuda_stream) for s in streams]
    meshes = [(capi.DeviceMesh(c, p.lowpoly), capi.DeviceMesh(c, p.dense)) for c, p in zip(ctxs, pairs)]
    outs = [torch.empty((p.res, p.res, 3), dtype=torch.uint8, device="cuda") for p in pairs]
    stats = [capi.MfBakeStats() for _ in range(k)]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    main = torch.cuda.current_stream()
    pool = cf.ThreadPoolExecutor(max_workers=k)

    def one(i):
        c, (lo, hi), p = ctxs[i], meshes[i], pairs[i]
        capi.check(c.lib.mf_bake_normal_map_dev(c.h, lo.h, hi.h, p.res, p.bbox_diagonal, p.max_distance_fraction,
                                                4, 0, p.res, outs[i].data_ptr(), stats[i]))

    def batch():
        ev = torch.cuda.Event()
        ev.record(main)
        for s in streams:
            s.wait_event(ev)
        list(pool.map(one, range(k)))
        for s in streams:
            main.wait_stream(s)

    ms, clocks = timed_steps(d, batch, args.steps, args.warmup, main, flush, d.device)
    nv = sum(s.valid_texels for s in stats)
    launches = args.steps * k * launches_per_bake(ctxs[0], lambda: one(0))
    ms, = d.max(ms)
    nv, = d.sum(nv)
    pool.shutdown()
    for c in ctxs:
        c.synchronize()
    if d.rank != 0:
        return None
    out = {"metric": METRICS.get(name, METRIC), "value": nv / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (deterministic geodesic blob pairs, one seed per asset)",
           "config": config_dict(name, pairs[0], "batch", world, k, seed=fx.CONFIGS[name]["seed"]),
           "assets_per_gpu": k, "assets_total": k * world, "ms_per_asset": ms / k,
           "ms_per_64_assets": ms * 64.0 / (k * world),
           "gpu_launches": launches, "clocks": clocks}
    if not as_line:
        out = {k_: v for k_, v in out.items() if k_ not in ("higher_is_better", "vs_baseline", "dtype", "data")}
    return out


def launches_per_bake(ctx, step):
    """Kernels one bake launches (counted on an eager run)."""
    before = ctx.launches
    ctx.set_timing(True)  # timing forces the eager path
    step()
    ctx.set_timing(False)
    return ctx.launches - before


def _pinned_pair(pair):
    import torch

    from paper_2605_26137_b200.mesh import TriangleMesh

    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    lo, hi = pair.lowpoly, pair.dense
    lo_p = TriangleMesh(pinned(lo.positions), pinned(lo.faces), uvs=pinned(lo.uvs), face_uvs=pinned(lo.face_uvs))
    hi_p = TriangleMesh(pinned(hi.positions), pinned(hi.faces))
    h2d = sum(a.nbytes for a in (lo_p.positions, lo_p.faces, lo_p.uvs, lo_p.face_uvs, hi_p.positions, hi_p.faces))
    return lo_p, hi_p, h2d


def _time_calls(call, stream, steps):
    import torch
    times = []
    for _ in range(steps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        call()
        e.record(stream)
        e.synchronize()
        times.append(s.elapsed_time(e))
    return times


def run_e2e(args, d, ctx, pair):
    """mf_bake_normal_map from host buffers: pinned (the headline e2e) and
    pageable numpy arrays (what a drop-in caller's std::vectors are)."""
    import ctypes

    import torch

    from paper_2605_26137_b200 import capi

    lo_p, hi_p, h2d = _pinned_pair(pair)
    res = pair.res
    out = torch.empty((res, res, 3), dtype=torch.uint8).pin_memory().numpy()
    out_pg = np.empty((res, res, 3), np.uint8)
    st = capi.MfBakeStats()
    stream = torch.cuda.current_stream()

    def call_with(lv, hv, o):
        def call():
            capi.check(ctx.lib.mf_bake_normal_map(ctx.h, ctypes.byref(lv), ctypes.byref(hv), res,
                                                  pair.bbox_diagonal, pair.max_distance_fraction, 4,
                                                  ctypes.c_void_p(o.ctypes.data), None, None, ctypes.byref(st)))
        return call

    steps = max(10, min(3 * args.steps, 30))
    res_out = {}
    for tag, (lm, hm, o) in {"pinned": (lo_p, hi_p, out), "pageable": (pair.lowpoly, pair.dense, out_pg)}.items():
        lv, hv = lm.view(), hm.view()
        call = call_with(lv, hv, o)
        for _ in range(5):  # eager, graph capture, replays
            call()
        torch.cuda.synchronize()
        times = _time_calls(call, stream, steps)
        ms, = d.max(statistics.mean(times))
        nv, = d.sum(st.valid_texels)
        res_out[tag] = {"value": nv / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
                        "ms_median": statistics.median(times), "ms_min": min(times), "steps": steps}
    assert np.array_equal(out, out_pg)
    e2e = dict(res_out["pinned"])
    api = run_e2e_api(pair, steps) if d.world == 1 else None
    e2e.update({"h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(out.nbytes),
                "call": "mf_bake_normal_map (host buffers, pinned) via ctypes",
                "pageable": dict(res_out["pageable"], call="mf_bake_normal_map from pageable numpy arrays "
                                                           "(a drop-in caller's std::vector data)")})
    if api is not None:
        e2e["api"] = api
    return e2e


def run_e2e_api(pair, steps):
    """The reference-facing C++ API end to end (tools/bench_api.cpp through
    libmeshforge_b200): TriangleMesh std::vectors in, ImageU8 out, wall clock,
    the fused meshforge::bakeNormalMap and the reference's three-call
    composition (each call round-trips its G-buffer / image through the host)."""
    import tempfile
    exe = os.path.join(ROOT, "build", "bench_api")
    if not os.path.exists(exe):
        return {"unavailable": f"{exe} not built"}
    with tempfile.TemporaryDirectory() as tmp:
        lo, hi = pair.lowpoly, pair.dense
        for name, a, dt in (("lo_pos.f64", lo.positions, np.float64), ("lo_faces.i32", lo.faces, np.int32),
                            ("lo_uvs.f64", lo.uvs, np.float64), ("lo_fuv.i32", lo.face_uvs, np.int32),
                            ("hi_pos.f64", hi.positions, np.float64), ("hi_faces.i32", hi.faces, np.int32)):
            np.ascontiguousarray(a, dtype=dt).tofile(os.path.join(tmp, name))
        p = subprocess.run([exe, tmp, str(pair.res), repr(pair.bbox_diagonal), repr(pair.max_distance_fraction),
                            "4", "3", str(steps)], capture_output=True, text=True, timeout=600)
    if p.returncode != 0:
        return {"unavailable": (p.stderr or p.stdout)[-300:]}
    r = json.loads(p.stdout.strip().splitlines()[-1])
    nv = _n_valid(pair)
    r.update({"value": nv / (r["fused_ms_mean"] * 1e-3), "unit": UNIT,
              "three_call_value": nv / (r["three_call_ms_mean"] * 1e-3),
              "call": "meshforge::bakeNormalMap (C++ API, pageable std::vector meshes, ImageU8 out; wall clock) "
                      "and dilateSeams(transferNormals(rasterizeGBuffer(lo, res), hi, diag, frac), g, 4)"})
    return r


def run_e2e_shard(args, d, ctx, pair, ranges, peer, gather):
    """Sharded bake end to end through the public ABI, per rank and step: the
    H2D upload + device validation of both meshes from pinned host memory
    (mf_mesh_upload), the rank's row slab with its gather into every rank's
    atlas, a barrier, and the D2H of the assembled atlas into pinned memory."""
    import ctypes

    import torch

    from paper_2605_26137_b200 import capi, sharding

    lo_p, hi_p, h2d = _pinned_pair(pair)
    res = pair.res
    b, e = ranges[d.rank]
    out = torch.empty((res, res, 3), dtype=torch.uint8).pin_memory()
    rows_max = max(hi_ - lo_ for lo_, hi_ in ranges)
    slab = torch.empty((rows_max, res, 3), dtype=torch.uint8, device="cuda")
    rgb = torch.empty((res, res, 3), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def call():
        lo = capi.DeviceMesh(ctx, lo_p)
        hi = capi.DeviceMesh(ctx, hi_p)
        if peer is not None:
            capi.check(ctx.lib.mf_bake_normal_map_dev_publish(ctx.h, lo.h, hi.h, res, pair.bbox_diagonal,
                                                              pair.max_distance_fraction, 4, b, e, peer.dst,
                                                              peer.n, None))
            d.barrier()
            out.copy_(peer.atlas, non_blocking=True)
        else:
            capi.check(ctx.lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, res, pair.bbox_diagonal,
                                                      pair.max_distance_fraction, 4, b, e, slab.data_ptr(), None))
            if d.backend == "nccl":
                g = [torch.empty_like(slab) for _ in ranges]
                torch.distributed.all_gather(g, slab)
                rgb.copy_(sharding.assemble(g, ranges))
            else:
                g = [torch.empty_like(slab, device="cpu") for _ in ranges]
                torch.distributed.all_gather(g, slab.cpu())
                rgb.copy_(sharding.assemble(g, ranges).to("cuda"))
            out.copy_(rgb, non_blocking=True)
        lo.close()
        hi.close()

    for _ in range(4):
        call()
    torch.cuda.synchronize()
    d.barrier()
    steps = max(5, min(args.steps, 20))
    times = _time_calls(call, stream, steps)
    ms, = d.max(statistics.mean(times))
    return {"value": float(_n_valid(pair)) / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "ms_median": statistics.median(times), "steps": steps, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(out.numel()),
            "call": "per rank: mf_mesh_upload x2 (pinned host meshes) + sharded bake + gather + barrier + "
                    "D2H of the whole atlas; bytes are per rank"}


# ----------------------------------------------------------------------------- CPU reference
def _reference_lib():
    from oracle import bindings
    if bindings.ref_available():
        return bindings.ref(), "reference"
    return bindings.port(), "port"


def cpu_reference_bake(pair, time_bvh=False, debug=False):
    lib, kind = _reference_lib()
    t0 = time.perf_counter()
    if kind == "reference":
        r = lib.bake(pair.lowpoly, pair.dense, pair.res, pair.bbox_diagonal, pair.max_distance_fraction, 4,
                     time_bvh=time_bvh, debug=debug)
    else:
        r = lib.bake(pair.lowpoly, pair.dense, pair.res, pair.bbox_diagonal, pair.max_distance_fraction, 4,
                     debug=debug)
    wall = time.perf_counter() - t0
    return r, wall, kind, r.get("n_valid")


def cores():
    lib, kind = _reference_lib()
    if kind == "reference":
        return lib.hardware_threads()
    return os.cpu_count() or 1


def atlas_parity(pair, ctx, r, gpu_rgb):
    """The GPU atlas of the timed run against the reference's (same inputs):
    RGB8 mismatches (count, max LSB, and how many are NOT explained by the
    .5-boundary rule of SURVEY §8c), plus hit faces of a GPU debug bake
    against the reference replica's (Appendix D)."""
    from paper_2605_26137_b200 import meshforge as mf
    ref_rgb = r["rgb"].reshape(-1, 3).astype(np.int32)
    g = gpu_rgb.reshape(-1, 3).astype(np.int32)
    diff = np.abs(g - ref_rgb)
    bad = np.argwhere(diff > 0)
    out = {"texels": int(ref_rgb.shape[0]), "rgb_mismatch_texels": int((diff.max(1) > 0).sum()),
           "rgb_max_lsb": int(diff.max()) if diff.size else 0}
    ts = r.get("ts")
    if ts is not None:
        v = (ts.reshape(-1, 3)[bad[:, 0], bad[:, 1]] + 1.0) * 127.5
        near = np.abs(v - np.floor(v) - 0.5) <= 1e-3 * 127.5
        out["rgb_outside_rule"] = int(((diff[bad[:, 0], bad[:, 1]] > 1) | ~near).sum())
    if r.get("face") is not None and ctx is not None:
        dbg = mf.bake_normal_map(pair.lowpoly, pair.dense, pair.res, pair.bbox_diagonal,
                                 pair.max_distance_fraction, 4, debug=True, ctx=ctx)
        out["face_mismatch"] = int((dbg["face"] != r["face"]).sum())
        out["queries"] = int((r["face"] != -1).sum())
        out["debug_rgb_equals_timed"] = bool(np.array_equal(dbg["rgb"].reshape(-1, 3), gpu_rgb.reshape(-1, 3)))
        if ts is not None:
            out["ts_max_abs_diff"] = float(np.abs(dbg["ts"] - ts).max())
    out["ok"] = (out["rgb_max_lsb"] <= 1 and out.get("rgb_outside_rule", 0) == 0
                 and out.get("face_mismatch", 0) == 0)
    return out


def cpu_baseline(pair, name, runs=5, ctx=None, gpu_rgb=None):
    """The reference's CPU bake (rasterizeGBuffer + transferNormals + dilateSeams,
    as test_bake.cpp:205-206 composes it) on the box's host cores, median of
    `runs` full bakes (~8 s at B), with a standalone Bvh(hi) build
    timed beside it (not part of the total: transferNormals builds its own).
    The first run also returns per-texel hit faces and ts (the reference
    replica, run after the timed stock chain) and its atlas is diffed against
    the GPU's (`parity`)."""
    runs_t = []
    parity = None
    bvh_s = 0.0
    for i in range(runs):
        dbg = i == 0 and gpu_rgb is not None
        r, wall, kind, _ = cpu_reference_bake(pair, time_bvh=(i == 0), debug=dbg)
        times = r.get("times") or {}
        if i == 0:
            bvh_s = times.get("bvh", 0.0) or 0.0
        if dbg:
            parity = atlas_parity(pair, ctx, r, gpu_rgb)
        runs_t.append((times.get("total", wall) or wall, times))
        del r
    runs_t.sort(key=lambda x: x[0])
    t, times = runs_t[len(runs_t) // 2]
    times = dict(times, bvh=bvh_s)
    n_valid = _n_valid(pair)
    return {"value": n_valid / t, "unit": UNIT, "cores": cores(), "kind": kind,
            "sample": f"median of {runs} full {name} bakes (raster + transfer incl. its normals and BVH build + "
                      f"dilate r=4), {t:.3f} s; median run's stages s: "
                      + ", ".join(f"{k} {v:.3f}" for k, v in times.items() if k != "bvh")
                      + f"; standalone Bvh(hi) build {bvh_s:.3f} s (outside the total)",
            "threads_note": "std::thread::hardware_concurrency() threads in the transfer loop only, "
                            "raster/BVH/dilate single-threaded, exactly as shipped (core/parallel.h)",
            "parity": parity}


_NV_CACHE = {}


def n_queries_full(name, pair):
    try:
        with open(CONSTANTS) as f:
            return int(json.load(f)[name]["n_queries"])
    except (OSError, KeyError):
        return _n_valid(pair)


def _n_valid(pair):
    key = id(pair)
    if key not in _NV_CACHE:
        try:
            with open(CONSTANTS) as f:
                c = json.load(f)
            _NV_CACHE[key] = int(c[pair.name]["n_valid"])
        except (OSError, KeyError):
            from oracle import bindings
            g = bindings.port().raster_gbuffer(pair.lowpoly, pair.res)
            _NV_CACHE[key] = int(g.valid.sum())
    return _NV_CACHE[key]


def run_reference(args, mode, name):
    """The reference's own CPU bake on the host cores (rank 0 only), on this
    arm's workload and config dict. Each step is one full bake; the number of
    steps actually run is capped so the whole run stays within ~2.5 minutes
    (`steps` reports what ran, `steps_requested` what was asked)."""
    rank, _, world = dist_env()
    if rank != 0:
        return None
    from paper_2605_26137_b200 import fixtures as fx
    seed = fx.CONFIGS[name]["seed"]
    pair = fx.config_pair(name, seed=seed)
    n_valid = _n_valid(pair)
    budget_s = 150.0
    t_start = time.perf_counter()
    warm = min(args.warmup, 1)
    t_one = None
    for _ in range(warm):
        t0 = time.perf_counter()
        cpu_reference_bake(pair)
        t_one = time.perf_counter() - t0
    steps = args.steps
    if t_one:
        steps = max(1, min(args.steps, int((budget_s - (time.perf_counter() - t_start)) / t_one)))
    ts = []
    kind = None
    for _ in range(steps):
        r, wall, kind, _ = cpu_reference_bake(pair)
        times = r.get("times") or {}
        ts.append(times.get("total", wall) or wall)
    t = statistics.mean(ts)
    value = n_valid / t
    return {
        "metric": METRICS.get(name, METRIC), "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "steps_requested": args.steps, "warmup": warm, "warmup_requested": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong" if mode == "shard" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (same pair as --impl ours)",
        "config": config_dict(name, pair, mode, world, args.assets, seed=seed),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": kind,
                         "sample": f"one full {name} bake per step ({steps} steps), rasterizeGBuffer + "
                                   f"transferNormals (incl. its BVH build) + dilateSeams, rank 0 only",
                         "threads_note": "hardware_concurrency() threads in the transfer loop, the rest "
                                         "single-threaded as shipped (core/parallel.h)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def launch_selftest(args):
    """CPU check of the launcher (tests/test_bench_launch.py): every rank joins
    a gloo group and rank 0 prints the line shape with the group's size."""
    import torch.distributed as dist
    rank, _, world = dist_env()
    if "RANK" in os.environ:
        dist.init_process_group("gloo")
        import torch
        t = torch.ones(1)
        dist.all_reduce(t)
        world = int(t.item())
        dist.destroy_process_group()
    if rank != 0:
        return None
    mode, name = resolve(args, world)
    return {"metric": METRICS.get(name, METRIC), "n_gpus": world, "mode": mode, "config_name": name,
            "selftest": True}


def main():
    argv = sys.argv[1:]
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch(argv, args.gpus))
    _, _, world = dist_env()
    # (the reference arm is not re-launched: outside torchrun --gpus N still
    # selects the N-GPU workload)
    mode, name = resolve(args, world if "WORLD_SIZE" in os.environ else max(world, args.gpus))
    if args.launch_selftest:
        line = launch_selftest(args)
    elif args.impl == "reference":
        line = run_reference(args, mode, name)
    else:
        line = run_ours(args, mode, name)
    if line is not None:
        s = json.dumps(line)
        print(s, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(s + "\n")


if __name__ == "__main__":
    main()
