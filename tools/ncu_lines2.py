#!/usr/bin/env python
"""Per-source-line warp instructions and SIMT efficiency from
`ncu --page source --csv --print-source cuda,sass` (source-line rows)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
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
        d = dict(zip(hdr[2:], r[2:]))
        try:
            ins = int(r[7] or 0)
            thr = int(r[8] or 0)
            s = int(r[4] or 0)
        except ValueError:
            continue
        if ins:
            data.append((ins, thr, s, fname, r[0], r[1].strip()[:80]))
tot = sum(x[0] for x in data) or 1
tot_t = sum(x[1] for x in data) or 1
tot_s = sum(x[2] for x in data) or 1
print(f"warp instr {tot}, thread instr {tot_t}, SIMT eff {tot_t / tot / 32:.2f}")
for ins, thr, s, f, l, src in sorted(data, reverse=True)[:top]:
    print(f"inst {ins / tot * 100:5.1f}%  eff {thr / ins / 32:4.2f}  stall {s / tot_s * 100:5.1f}%  {f}:{l:<5} {src}")
