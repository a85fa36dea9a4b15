#!/usr/bin/env python
"""Summarise `ncu --page source --csv --print-source cuda,sass`: top source lines by warp
stall samples and by executed warp instructions (lines aggregate their SASS)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = sys.argv[3] if len(sys.argv) > 3 else "stall"
fname, hdr, data = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 4 and r[2] == "-":
        try:
            s = int(r[4] or 0)
            ins = int(r[7] or 0)
        except ValueError:
            continue
        if s or ins:
            data.append((s if key == "stall" else ins, s, ins, fname, r[0], r[1].strip()[:90]))
tot_s = sum(x[1] for x in data) or 1
tot_i = sum(x[2] for x in data) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for _, s, ins, f, l, src in sorted(data, reverse=True)[:top]:
    print(f"stall {s / tot_s * 100:5.1f}%  inst {ins / tot_i * 100:5.1f}%  {f}:{l:<5} {src}")
