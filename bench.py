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
    ap.add_argument("--json-out", default=None)
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

    def step(stats=None):
        if shard_ranges is None:
            capi.check(lib.mf_bake_normal_map_dev(ctx.h, lo.h, hi.h, res, diag, frac, 4, 0, res,
                                                  rgb.data_ptr(), stats))
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
    roofline = None
    if alg_bytes is not None:
        achieved = alg_bytes / (ms_transfer * 1e-3) / 1e9
        traffic, traffic_src = transfer_traffic()
        roofline = {"bound": "hbm", "kernel": "k_transfer_t (closest-point traversal + encode)",
                    "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                    "peak_source": peak_src,
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
                   "parallelism": (f"rows x{world} (one atlas, valid-balanced row slabs, NCCL all-gather)"
                                   if shard_ranges else f"assets x{world} (one asset per GPU, no collective)"),
                   "l2": "flushed between timed steps (256 MiB write, outside the per-step events)",
                   "seed": fx.CONFIGS[name]["seed"]},
        "rays_per_s": agg_nq / (t_xfer_max * 1e-3),
        "n_valid_texels": n_valid, "n_queries": n_queries, "hits": hits,
        "stage_ms": {k: round(statistics.mean(v), 4) for k, v in stage.items()},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks,
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

    for _ in range(2):
        call()
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 10))
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
    return {"value": nv / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "call": "mf_bake_normal_map (host buffers, pinned) via ctypes"}


# ----------------------------------------------------------------------------- CPU reference
def _reference_lib():
    from oracle import bindings
    if bindings.ref_available():
        return bindings.ref(), "reference"
    return bindings.port(), "port"


def cpu_reference_bake(pair):
    lib, kind = _reference_lib()
    t0 = time.perf_counter()
    r = lib.bake(pair.lowpoly, pair.dense, pair.res, pair.bbox_diagonal, pair.max_distance_fraction, 4)
    wall = time.perf_counter() - t0
    return r, wall, kind, r.get("n_valid")


def cores():
    lib, kind = _reference_lib()
    if kind == "reference":
        return lib.hardware_threads()
    return os.cpu_count() or 1


def cpu_baseline(pair, name):
    """The reference's CPU bake (rasterizeGBuffer + transferNormals + dilateSeams,
    as test_bake.cpp:205-206 composes it) on the box's host cores: one full
    config bake is the bounded sample (~5-20 s)."""
    r, wall, kind, _ = cpu_reference_bake(pair)
    times = r.get("times") or {}
    t = times.get("total", wall) or wall
    n_valid = _n_valid(pair)
    return {"value": n_valid / t, "unit": UNIT, "cores": cores(), "kind": kind,
            "sample": f"one full {name} bake (raster + transfer incl. its BVH build + dilate r=4), "
                      f"{t:.2f} s; stages s: " + ", ".join(f"{k} {v:.3f}" for k, v in times.items()),
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
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        s = json.dumps(line)
        print(s, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(s + "\n")


if __name__ == "__main__":
    main()
