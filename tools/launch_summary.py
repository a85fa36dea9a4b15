#!/usr/bin/env python
"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
skip_gen = "--all" not in sys.argv
hdr, recs = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        recs.append(dict(zip(hdr, r)))
per = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for d in recs:
    name = d["Kernel Name"].split("(")[0].replace("rlg::", "").replace("(anonymous namespace)::", "")
    if skip_gen and "generate" in name:
        continue
    key = (d["ID"], name)
    per[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (lid, name), m in per.items():
    a = agg[name]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0)
    a[3] += m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':28s} {'n':>4s} {'mean us':>10s} {'share':>7s} {'GB/s':>8s} {'MB rd/launch':>13s} {'MB wr/launch':>13s}")
for name, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
    gbs = (rd + wr) / t if t else 0  # bytes/ns = GB/s
    print(f"{name:28s} {n:4d} {t / n / 1e3:10.1f} {t / tot * 100:6.1f}% {gbs:8.0f} {rd / n / 1e6:13.1f} {wr / n / 1e6:13.1f}")
print(f"total {tot / 1e6:.3f} ms over {sum(a[0] for a in agg.values())} launches")
