#!/usr/bin/env python
"""Summarise tools/prof_driver.py --sweep output (per-image ms per phase)."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
print("d     g   analyze  merge    emit     total(ms/img)  Gpx/s")
for r in rows:
    if r["g"] in (1, 4, 16) and round(r["d"] * 20) % 2 == 0:
        print(f"{r['d']:.2f} {r['g']:3d} {r['analyze']:.4f}  {r['merge']:.4f}  {r['emit']:.4f}  {r['total']:.4f}  {r['gpx']:8.1f}")
tot = sum(r["total"] for r in rows)
parts = {k: sum(r[k] for r in rows) for k in ("analyze", "merge", "emit")}
print("sum per-image ms %.3f  -> %.1f Gpx/s (separate batches)" % (tot, len(rows) * 4194304 / (tot / 1e3) / 1e9))
print({k: round(v, 3) for k, v in parts.items()})
by_g = {}
for r in rows:
    by_g[r["g"]] = by_g.get(r["g"], 0) + r["total"]
print({g: round(v, 3) for g, v in by_g.items()})
