#!/usr/bin/env python
"""Executed warp instructions of an `ncu --page source --csv --print-source cuda,sass` export
summed over source-line ranges: ncu_ranges.py <csv> file:a-b[:name] ..."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname, hdr, per = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 7 and r[2] == "-":
        try:
            per[(fname, int(r[0]))] = per.get((fname, int(r[0])), 0) + int(r[7] or 0)
        except ValueError:
            pass
tot = sum(per.values()) or 1
done = 0
for spec in sys.argv[2:]:
    parts = spec.split(":")
    f, (a, b) = parts[0], map(int, parts[1].split("-"))
    name = parts[2] if len(parts) > 2 else ""
    s = sum(v for (ff, l), v in per.items() if ff == f and a <= l <= b)
    done += s
    print(f"{s / tot * 100:5.1f}%  {f}:{a}-{b} {name}")
print(f"{(tot - done) / tot * 100:5.1f}%  other; total {tot}")
others = sorted(((v, k) for k, v in per.items()), reverse=True)
