#!/usr/bin/env python
"""Per-kernel table + JSON from the raw metric CSVs of tools/ncu_all.sh
(`ncu --metrics <ncu_summary.METRICS> --csv --page raw`): first launch of
each kernel per part.

  python tools/ncu_csv_summary.py TAG [part=csv ...]
  e.g. python tools/ncu_csv_summary.py r02o bake=gpurun_out/r02o_bake_metrics.csv \
       secondary=gpurun_out/r02o_secondary_metrics.csv E=gpurun_out/r02o_E_metrics.csv
writes profiles/TAG_ncu_all_kernels.{txt,json}."""
from __future__ import annotations

import csv
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import METRICS  # noqa: E402


def rows(path):
    text = open(path, errors="replace").read()
    start = text.find('"ID"')
    rd = list(csv.reader(io.StringIO(text[start:])))
    head, units, body = rd[0], rd[1], rd[2:]
    idx = {h: i for i, h in enumerate(head)}
    out, seen = [], set()
    for r in body:
        if len(r) != len(head):
            continue
        name = r[idx["Kernel Name"]]
        short = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "").replace("mfb::", "").replace("void ", "")
        short = short.split("(")[0]
        if short in seen:
            continue
        seen.add(short)
        d = {"kernel": short}
        for m, key in METRICS.items():
            if m not in idx:
                continue
            v = r[idx[m]].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[idx[m]]
            scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6, "nsecond": 1.0}
            d[key] = x * scale.get(u, 1.0)
        d["dram_bytes"] = d.get("dram_read_bytes", 0.0) + d.get("dram_write_bytes", 0.0)
        out.append(d)
    return out


def main():
    tag = sys.argv[1]
    parts = dict(a.split("=", 1) for a in sys.argv[2:])
    res = {"source": ", ".join(parts.values()) + " (ncu --metrics <tools/ncu_summary.py METRICS> --clock-control "
                                                  "none; tools/ncu_all.sh, tools/round_profile.sh)"}
    lines = [f"# {tag}: ncu counters, cold caches, serialised launches (first launch of each kernel per part)",
             "part      kernel                                    us   DRAM MB DRAM GB/s  L2 GB/s   occ% issue% "
             "thr/in  L1hit  L2hit"]
    for part, path in parts.items():
        ks = rows(path)
        res[part] = ks
        for d in ks:
            us = d.get("duration_ns", 0.0) / 1e3
            dram = d["dram_bytes"]
            l2 = d.get("l2_sectors", 0.0) * 32
            lines.append(f"{part:<9} {d['kernel'][:40]:<40} {us:7.1f} {dram / 1e6:9.1f} {dram / max(us, 1e-9) / 1e3:9.0f} "
                         f"{l2 / max(us, 1e-9) / 1e3:8.0f} {d.get('achieved_occupancy_pct', 0):6.1f} "
                         f"{d.get('issue_active_pct', 0):6.1f} {d.get('threads_per_instruction', 0):6.1f} "
                         f"{d.get('l1_hit_pct', 0):6.1f} {d.get('l2_hit_pct', 0):6.1f}")
    os.makedirs("profiles", exist_ok=True)
    with open(f"profiles/{tag}_ncu_all_kernels.json", "w") as f:
        json.dump(res, f, indent=1)
        f.write("\n")
    with open(f"profiles/{tag}_ncu_all_kernels.txt", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
