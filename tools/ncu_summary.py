#!/usr/bin/env python
"""Summarise ncu artefacts into profiles/ (committed evidence).

  python tools/ncu_summary.py launches gpurun_out/r01_launches.csv > profiles/r01_launches.txt
  python tools/ncu_summary.py full gpurun_out/r01_prof_k_transfer.ncu-rep [--json profiles/r01_k_transfer.json]

`launches` aggregates a `--metrics gpu__time_duration.sum` launch list per
kernel per bake (cold-cache, serialised: compare shares, not absolutes).
`full` extracts duration, DRAM/L2/L1 bytes and rates, occupancy, issue
activity, SIMT width and the stall mix of one `--set full` capture.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "lts__t_sectors.sum": "l2_sectors",
    "l1tex__t_sectors.sum": "l1_sectors",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_instruction",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_executed_pipe_fp64.sum": "fp64_pipe_instructions",
}


def _kname(n: str) -> str:
    """Short kernel name: drop `void`, namespaces (ncu prints the anonymous one
    as `<unnamed>`) and the argument list; keep template arguments."""
    n = n.replace("(anonymous namespace)", "<unnamed>").replace("void ", "").split("(")[0]
    if n.startswith(("mfb::", "unnamed>::")):
        n = n.rsplit("::", 1)[-1]
    return n


def _num(v: str) -> float:
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = _num(r[vi])
        unit = r[ui]
        us = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
        name = _kname(r[ki])
        agg.setdefault(name, []).append(us)
    ref = [k for k in agg if "k_transfer" in k]
    bakes = len(agg[ref[0]]) if ref else 1
    total = sum(sum(v) for v in agg.values()) / bakes
    out = io.StringIO()
    out.write(f"# {path}: {bakes} bakes, {total:.1f} us of kernel time per bake (cold, serialised)\n")
    out.write(f"{'us/bake':>10} {'share':>6} {'launches':>8}  kernel\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        s = sum(v) / bakes
        out.write(f"{s:10.1f} {100 * s / total:5.1f}% {len(v) / bakes:8.1f}  {k}\n")
    return out.getvalue()


def full(path: str) -> dict:
    if path.endswith(".csv"):  # `ncu --metrics ... --csv --page raw --log-file` output
        raw = open(path).read()
        raw = raw[raw.index('"ID"'):] if '"ID"' in raw else raw
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    header, units = rows[0], rows[1]
    results = []
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6,
             "s": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3,
             "MB": 1e6, "GB": 1e9}
    unit_of = dict(zip(header, units))
    for r in rows[2:]:
        d = dict(zip(header, r))
        res = {"kernel": _kname(d.get("Kernel Name", ""))}
        for m, key in METRICS.items():
            if m in d:
                res[key] = _num(d[m]) * scale.get(unit_of.get(m, ""), 1.0)
        if "dram_read_bytes" in res and "dram_write_bytes" in res:
            res["dram_bytes"] = res["dram_read_bytes"] + res["dram_write_bytes"]
        results.append(res)
    return {"source": path, "launches": results}


def main():
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches":
        print(launches(path), end="")
    else:
        s = full(path)
        text = json.dumps(s, indent=1)
        if "--json" in sys.argv:
            with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
                f.write(text + "\n")
        print(text)


if __name__ == "__main__":
    main()
