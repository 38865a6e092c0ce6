#!/usr/bin/env python
"""Per-CUDA-source-line stall samples and instruction counts from an ncu
`--page source --print-source cuda,sass --csv` export (lines with a Line No)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
out = []; fname = ''
hdr = None
for r in rows:
    if r and r[0] == 'File Path': fname = r[1].split('/')[-1]
    if r and r[0] == 'Line No': hdr = r; continue
    if hdr and r and r[0] and r[0] != 'Line No' and r[0].isdigit():
        try:
            s = int(r[4] or 0); n = int(r[7] or 0)
        except ValueError:
            continue
        out.append((s, n, f'{fname}:{r[0]}', r[1].strip()[:110]))
tot = sum(o[0] for o in out) or 1
out.sort(reverse=True)
for s, n, loc, src in out[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f'{s/tot*100:5.1f}% {n:>10d} {loc:22s} {src}')
