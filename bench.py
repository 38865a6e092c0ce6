#!/usr/bin/env python
"""Benchmark: baked texels/s (+ BVH rays/s) of the fused B200 normal bake.

Workload (BASELINE.json configs[1], "config B"): synthetic geodesic pair,
dense G(224) = 1,003,520 faces -> lowpoly G(32) = 20,480 faces with a 20-chart
UV atlas, 2048^2 atlas, maxDistanceFraction 0.01, dilation radius 4.
One step = one whole bake: dense vertex normals + LBVH build + lowpoly wedge
frames/reliability + raster + closest-point transfer + dilation, i.e.
dilateSeams(transferNormals(rasterizeGBuffer(lo), hi, diag), g, 4) of the
reference (test_bake.cpp:205-206), with the meshes already resident in HBM.

`value`  = N_v / t_step   (baked texels/s, device time, CUDA events)
`e2e`    = the same bake through the host-buffer C ABI call
           (mf_bake_normal_map) from pinned host memory: H2D of both meshes,
           device validation, bake, D2H of the RGB8 atlas inside the timing.
Multi-GPU (torchrun, N ranks): each rank bakes its own asset (seed 7 + rank),
no data-path collective (batches of independent assets, SURVEY §8e config D
style) -> "scaling": "weak"; value = sum_r N_v(r) / max_r t.

`--impl reference` times the reference's own CPU implementation (the
reference TUs compiled in place, oracle/_ref/libmfref.so; the C restatement
oracle/build/liboracle.so if that is absent) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="B")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rays", action="store_true", help="skip the secondary BVH rays/s metrics")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--assets", type=int, default=1,
                    help="independent assets baked concurrently per GPU (config D: 8), one context + stream + "
                         "host thread each")
    ap.add_argument("--gather", choices=["nccl", "peer"], default="peer",
                    help="--shard: atlas gather by NCCL all-gather, or by the dilation kernel storing its rows "
                         "into every rank's atlas over CUDA IPC peer memory (mf_bake_normal_map_dev_publish)")
    ap.add_argument("--shard", action="store_true",
                    help="N>1: row-shard ONE atlas across ranks + NCCL all-gather (strong scaling) "
                         "instead of one asset per rank")
    return ap.parse_args()


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


def stage_rooflines(pair, stage, n_queries, counters, hbm, peaks):
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
        "dilate": row(7 * res * res, stage["ms_dilate"], hbm, note="7 B x res^2"),
    }
    if counters:
        out["transfer_l2"] = row(counters["bytes_per_query"] * n_queries, stage["ms_transfer"],
                                 peaks.get("l2_read_gbs"), note="W_q x N_q against the measured L2 read bandwidth")
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


def transfer_traffic():
    """dram__bytes_read + dram__bytes_write of the transfer kernel from the
    committed `ncu --set full` capture summary (profiles/k_transfer_ncu.json)."""
    try:
        with open(TRAFFIC) as f:
            d = json.load(f)
        launch = next(x for x in d["launches"] if "k_transfer" in x["kernel"])
        return float(launch["dram_bytes"]), d.get("source")
    except (OSError, KeyError, StopIteration, ValueError):
        return None, None


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
def run_ours(args):
    import torch

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    distributed = "RANK" in os.environ  # launched by torchrun (any world size)
    if distributed:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2605_26137_b200 import capi, fixtures as fx

    name = args.config
    pair = fx.config_pair(name, seed=fx.CONFIGS[name]["seed"] + (0 if args.shard else rank))
    res = pair.res
    stream = torch.cuda.current_stream()
    ctx = capi.Context(local_rank, stream.cuda_stream)
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
    if args.shard and distributed:
        # one atlas, rows balanced by valid texels, all-gathered
        import ctypes
        from paper_2605_26137_b200 import sharding
        counts = np.zeros(res, np.int64)
        capi.check(lib.mf_coverage_rows(ctx.h, lo.h, res, ctypes.c_void_p(counts.ctypes.data)))
        shard_ranges = sharding.balanced_row_ranges(counts, world)
        row_b, row_e = shard_ranges[rank]
        rows_max = max(e - b for b, e in shard_ranges)
        slab = torch.empty((rows_max, res, 3), dtype=torch.uint8, device="cuda")
        gathered = [torch.empty_like(slab) for _ in range(world)]
        peer = sharding.PeerAtlas(ctx, res) if args.gather == "peer" else None

    def step(stats=None):
        if shard_ranges is None:
            capi.check(lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, res, diag, frac, 4, 0, res,
                                                  rgb.data_ptr(), stats))
            return
        if peer is not None:  # rows stored into every rank's atlas by the dilation kernel
            capi.check(lib.mf_bake_normal_map_dev_publish(ctx.h, lo.h, hi.h, res, diag, frac, 4, row_b, row_e,
                                                          peer.dst, peer.n, stats))
            torch.distributed.barrier()
            return
        capi.check(lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, res, diag, frac, 4, row_b, row_e,
                                              slab.data_ptr(), stats))
        torch.distributed.all_gather(gathered, slab)
        rgb.copy_(sharding.assemble(gathered, shard_ranges))

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # timed region: per-step CUDA events on the launching stream, L2 flushed
    # (untimed) between steps. The library replays its captured CUDA graph of
    # the whole bake here (stage events are not meaningful inside a graph).
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = ctx.launches
    n_valid = n_queries = hits = 0
    if distributed:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            step(st)
            ends[i].record(stream)
            n_valid, n_queries, hits = st.valid_texels, st.queries, st.hits
        torch.cuda.synchronize()
    if distributed:
        torch.distributed.barrier()
    launches = ctx.launches - launches0
    if launches == 0:  # graph replays do not pass through the host launch counter
        launches = args.steps * launches_per_bake(ctx, step)
    # stage breakdown + the transfer kernel's own duration: the same bake run
    # eagerly with CUDA events around each stage on the launching stream
    ctx.set_timing(True)
    stage = {k: [] for k in ("ms_prepare", "ms_bvh", "ms_raster", "ms_transfer", "ms_dilate", "ms_total")}
    for i in range(max(3, min(args.steps, 10))):
        flush.zero_()
        step(st)
        d = st.as_dict()
        for k in stage:
            stage[k].append(d[k])
    ctx.set_timing(False)
    t_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    ms_step = t_ms / args.steps
    ms_transfer = statistics.mean(stage["ms_transfer"])

    # aggregate over ranks: max time, summed work
    agg_nv = n_valid
    agg_nq = n_queries
    t_max = ms_step
    t_xfer_max = ms_transfer
    if distributed:
        import torch.distributed as dist
        tt = torch.tensor([ms_step, ms_transfer], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        nn = torch.tensor([n_valid, n_queries], dtype=torch.float64, device="cuda")
        dist.all_reduce(nn, op=dist.ReduceOp.SUM)
        t_max, t_xfer_max = tt.tolist()
        agg_nv, agg_nq = nn.tolist()
        if shard_ranges is not None:  # slabs overlap by the dilation halo: count each texel once
            agg_nv, agg_nq = float(_n_valid(pair)), float(n_queries_full(name, pair))

    # secondary BVH metrics and the live L2 / FP64 peaks (rank 0)
    rays = bvh_rays(ctx, hi, pair, args.steps) if rank == 0 and not args.no_rays else None
    peaks = live_peaks(local_rank) if rank == 0 else {}

    # end-to-end through the host-buffer C ABI call (pinned host inputs/outputs)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, pair, world, distributed)

    if rank != 0:
        if distributed:
            torch.distributed.destroy_process_group()
        return None

    peak, peak_src = hbm_peak()
    alg_bytes, counters = transfer_algorithmic_bytes(name, n_queries, n_valid, res)
    stage_mean = {k: statistics.mean(v) for k, v in stage.items()}
    stages_rl = stage_rooflines(pair, stage_mean, n_queries, counters, peak, peaks)
    roofline = None
    if alg_bytes is not None:
        # the traversal's node/triangle bytes are served from L2
        # (its DRAM traffic, `traffic`, is ~5% of them), so its roofline is the
        # measured L2 read bandwidth; the HBM-relative figure is kept beside it.
        achieved = alg_bytes / (ms_transfer * 1e-3) / 1e9
        traffic, traffic_src = transfer_traffic()
        l2 = peaks.get("l2_read_gbs")
        roofline = {"bound": "l2" if l2 else "hbm", "kernel": "k_transfer_t (closest-point traversal + encode)",
                    "achieved": round(achieved, 1), "peak": l2 or peak, "unit": "GB/s",
                    "frac": round(achieved / (l2 or peak), 4), "traffic": traffic, "traffic_source": traffic_src,
                    "peak_source": ("measured live: L2 read bandwidth, tools/peaks.cu" if l2 else peak_src),
                    "hbm_peak": peak, "hbm_peak_source": peak_src, "frac_of_hbm": round(achieved / peak, 4),
                    "algorithmic_bytes_per_launch": alg_bytes, "ms_per_launch": round(ms_transfer, 4),
                    "per_query": counters}
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(pair, name)
    clocks = clk.summary()
    line = {
        "metric": METRICS.get(name, METRIC), "value": agg_nv / (t_max * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t_max,
        "higher_is_better": True, "scaling": "strong" if shard_ranges else "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (deterministic geodesic blob pair, Appendix B of SURVEY.md)",
        "config": {"workload": workload_desc(name, pair), "global_batch": 1 if shard_ranges else world,
                   "seq_len": None,
                   "parallelism": (f"rows x{world} (one atlas, valid-balanced row slabs, "
                                   f"{'peer-memory gather in the dilation kernel' if args.gather == 'peer' else 'NCCL all-gather'})"
                                   if shard_ranges else f"assets x{world} (one asset per GPU, no collective)"),
                   "l2": "flushed between timed steps (256 MiB write, outside the per-step events)",
                   "seed": fx.CONFIGS[name]["seed"]},
        "rays_per_s": agg_nq / (t_xfer_max * 1e-3),
        "n_valid_texels": n_valid, "n_queries": n_queries, "hits": hits,
        "stage_ms": {k: round(statistics.mean(v), 4) for k, v in stage.items()},
        "roofline": roofline, "stage_rooflines": stages_rl, "peaks": peaks, "bvh": rays,
        "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks,
    }
    if distributed:
        torch.distributed.destroy_process_group()
    return line


def run_batch(args):
    """K independent assets per GPU, each on its own
    context (own stream + side stream, own captured graph), driven by K host
    threads (ctypes drops the GIL in the call). One step = all K bakes;
    value = sum of valid texels over all assets of all ranks / max-rank time.
    Device time: one event on the launch stream that every asset stream waits
    on, and one after the launch stream joins every asset stream."""
    import concurrent.futures as cf

    import torch

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    distributed = "RANK" in os.environ
    if distributed:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2605_26137_b200 import capi, fixtures as fx

    name, k = args.config, args.assets
    base = fx.CONFIGS[name]["seed"] + rank * k
    pairs = [fx.config_pair(name, seed=base + i) for i in range(k)]
    streams = [torch.cuda.Stream() for _ in range(k)]
    ctxs = [capi.Context(local_rank, st.cuda_stream) for st in streams]
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
        for st in streams:
            st.wait_event(ev)
        list(pool.map(one, range(k)))
        for st in streams:
            main.wait_stream(st)

    for _ in range(max(args.warmup, 3)):
        batch()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if distributed:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = sum(c.launches for c in ctxs)
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(main)
            batch()
            ends[i].record(main)
        torch.cuda.synchronize()
    if distributed:
        torch.distributed.barrier()
    ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends)) / args.steps
    nv = sum(s.valid_texels for s in stats)
    launches = sum(c.launches for c in ctxs) - launches0
    if launches == 0:
        launches = args.steps * k * launches_per_bake(ctxs[0], lambda: one(0))
    if distributed:
        import torch.distributed as dist
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        nn = torch.tensor([nv], dtype=torch.float64, device="cuda")
        dist.all_reduce(nn, op=dist.ReduceOp.SUM)
        ms, nv = tt.item(), nn.item()
    pool.shutdown()
    if rank != 0:
        if distributed:
            torch.distributed.destroy_process_group()
        return None
    line = {
        "metric": METRICS.get(name, METRIC), "value": nv / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic geodesic blob pairs, one seed per asset)",
        "config": {"workload": workload_desc(name, pairs[0]) + f"; {k} assets per GPU (seeds {base}..{base + k - 1} "
                                                               f"on rank {rank})",
                   "global_batch": k * world, "seq_len": None,
                   "parallelism": f"assets x{k * world} ({k} per GPU on {k} streams, no collective)",
                   "l2": "flushed between timed steps (256 MiB write, outside the per-step events)"},
        "assets_per_gpu": k, "ms_per_asset": ms / k,
        "gpu_launches": launches, "clocks": clk.summary(),
    }
    if distributed:
        torch.distributed.destroy_process_group()
    return line


def launches_per_bake(ctx, step):
    """Kernels one bake launches (counted on an eager run)."""
    before = ctx.launches
    ctx.set_timing(True)  # timing forces the eager path
    step()
    ctx.set_timing(False)
    return ctx.launches - before


def run_e2e(args, ctx, pair, world, distributed=False):
    import ctypes
    import torch

    from paper_2605_26137_b200 import capi
    from paper_2605_26137_b200.mesh import TriangleMesh

    def pinned(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        return t.numpy()

    lo, hi = pair.lowpoly, pair.dense
    lo_p = TriangleMesh(pinned(lo.positions), pinned(lo.faces), uvs=pinned(lo.uvs), face_uvs=pinned(lo.face_uvs))
    hi_p = TriangleMesh(pinned(hi.positions), pinned(hi.faces))
    res = pair.res
    out = torch.empty((res, res, 3), dtype=torch.uint8).pin_memory().numpy()
    lv, hv = lo_p.view(), hi_p.view()
    h2d = sum(a.nbytes for a in (lo_p.positions, lo_p.faces, lo_p.uvs, lo_p.face_uvs, hi_p.positions, hi_p.faces))
    d2h = out.nbytes
    st = capi.MfBakeStats()
    stream = torch.cuda.current_stream()

    def call():
        capi.check(ctx.lib.mf_bake_normal_map(ctx.h, ctypes.byref(lv), ctypes.byref(hv), res, pair.bbox_diagonal,
                                              pair.max_distance_fraction, 4, ctypes.c_void_p(out.ctypes.data),
                                              None, None, ctypes.byref(st)))

    for _ in range(5):  # eager, graph capture, replays
        call()
    torch.cuda.synchronize()
    steps = max(10, min(3 * args.steps, 30))
    times = []
    for _ in range(steps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        call()
        e.record(stream)
        e.synchronize()
        times.append(s.elapsed_time(e))
    ms = statistics.mean(times)
    nv = st.valid_texels
    if distributed:
        import torch.distributed as dist
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        nn = torch.tensor([nv], dtype=torch.float64, device="cuda")
        dist.all_reduce(nn, op=dist.ReduceOp.SUM)
        ms = tt.item()
        nv = nn.item()
    return {"value": nv / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "ms_median": statistics.median(times),
            "ms_min": min(times), "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "call": "mf_bake_normal_map (host buffers, pinned) via ctypes"}


# ----------------------------------------------------------------------------- CPU reference
def _reference_lib():
    from oracle import bindings
    if bindings.ref_available():
        return bindings.ref(), "reference"
    return bindings.port(), "port"


def cpu_reference_bake(pair, time_bvh=False):
    lib, kind = _reference_lib()
    t0 = time.perf_counter()
    r = lib.bake(pair.lowpoly, pair.dense, pair.res, pair.bbox_diagonal, pair.max_distance_fraction, 4,
                 time_bvh=time_bvh)
    wall = time.perf_counter() - t0
    return r, wall, kind, r.get("n_valid")


def cores():
    lib, kind = _reference_lib()
    if kind == "reference":
        return lib.hardware_threads()
    return os.cpu_count() or 1


def cpu_baseline(pair, name, runs=5):
    """The reference's CPU bake (rasterizeGBuffer + transferNormals + dilateSeams,
    as test_bake.cpp:205-206 composes it) on the box's host cores, median of
    `runs` full bakes (~8 s at B), with a standalone Bvh(hi) build
    timed beside it (not part of the total: transferNormals builds its own)."""
    runs_t = []
    for i in range(runs):
        r, wall, kind, _ = cpu_reference_bake(pair, time_bvh=(i == 0))
        times = r.get("times") or {}
        if i == 0:
            bvh_s = times.get("bvh", 0.0)
        runs_t.append((times.get("total", wall) or wall, times))
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
                            "raster/BVH/dilate single-threaded, exactly as shipped (core/parallel.h)"}


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


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return None
    from paper_2605_26137_b200 import fixtures as fx
    name = args.config
    pair = fx.config_pair(name)
    n_valid = _n_valid(pair)
    for _ in range(args.warmup):
        cpu_reference_bake(pair)
    ts = []
    kind = None
    for _ in range(args.steps):
        r, wall, kind, _ = cpu_reference_bake(pair)
        times = r.get("times") or {}
        ts.append(times.get("total", wall) or wall)
    t = statistics.mean(ts)
    value = n_valid / t
    return {
        "metric": METRICS.get(name, METRIC), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (same pair as --impl ours)",
        "config": {"workload": workload_desc(name, pair), "global_batch": 1, "seq_len": None,
                   "parallelism": "host threads"},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": kind,
                         "sample": f"one full {name} bake per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    if args.impl == "reference":
        line = run_reference(args)
    elif args.assets > 1:
        line = run_batch(args)
    else:
        line = run_ours(args)
    if line is not None:
        s = json.dumps(line)
        print(s, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(s + "\n")


if __name__ == "__main__":
    main()
