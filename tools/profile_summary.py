#!/usr/bin/env python
"""Turn one round's ncu captures into the committed profiles/ artifacts.

  python tools/profile_summary.py --tag r01 --config cfg2 \
      --launches gpurun_out/launches_X.csv --full gpurun_out/prof_X.ncu-rep

writes profiles/<tag>_launches_<config>.csv (copy) and _summary.txt (per-kernel share of the
step, from the cold-cache serialised launch list), profiles/<tag>_ncu_full_<config>.txt (key
metrics of the tile kernels from the --set full capture) and profiles/traffic_<config>.json
(dram bytes per analyze/emit phase, read by bench.py's roofline.traffic).
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

FULL_METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "MB rd"),
    ("dram__bytes_write.sum", "MB wr"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occup %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "thr/inst"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp inst"),
]
PHASES = {"k_analyze": ("k_analyze", "k_analyze_m", "k_analyze_full"),
          "k_emit": ("k_emit", "k_emit_m", "k_emit_full")}


def short(name: str) -> str:
    return name.split("(")[0].replace("rlg::", "").replace("(anonymous namespace)::", "").strip()


def launch_summary(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hdr, recs = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            recs.append(dict(zip(hdr, r)))
    per = collections.defaultdict(dict)
    for d in recs:
        name = short(d["Kernel Name"])
        if "generate" in name or "rings" in name:
            continue
        per[(d["ID"], name)][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (_, name), m in per.items():
        a = agg[name]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0)
        a[3] += m.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    out = [f"{'kernel':28s} {'n':>4s} {'mean us':>10s} {'share':>7s} {'GB/s':>8s} {'MB rd/launch':>13s} {'MB wr/launch':>13s}"]
    for name, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = (rd + wr) / t if t else 0
        out.append(f"{name[:28]:28s} {n:4d} {t / n / 1e3:10.1f} {t / tot * 100:6.1f}% {gbs:8.0f} "
                   f"{rd / n / 1e6:13.1f} {wr / n / 1e6:13.1f}")
    out.append(f"total {tot / 1e6:.3f} ms over {sum(a[0] for a in agg.values())} launches "
               "(ncu --clock-control none, serialised, cold cache: shares, not absolute times)")
    return "\n".join(out)


def full_summary(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(m for m, _ in FULL_METRICS)], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(hdr)}
    table, traffic = [], collections.defaultdict(float)
    for r in rows[2:]:
        name = short(r[col["Kernel Name"]])
        vals = {}
        for m, _ in FULL_METRICS:
            if m not in col:
                continue
            v = float(r[col[m]].replace(",", "") or 0)
            u = units[col[m]]
            if m.startswith("dram__bytes"):
                v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
            if m == "gpu__time_duration.sum":
                v = v * {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)
            vals[m] = v
        table.append((r[col["ID"]], name, vals))
        for ph, members in PHASES.items():
            if name in members:
                traffic[ph] += (vals.get("dram__bytes_read.sum", 0) + vals.get("dram__bytes_write.sum", 0)) * 1e6
    out = [f"{'id':>3s} {'kernel':16s} " + " ".join(f"{lab:>10s}" for _, lab in FULL_METRICS)]
    for lid, name, vals in table:
        out.append(f"{lid:>3s} {name[:16]:16s} " + " ".join(
            f"{vals.get(m, float('nan')):10.1f}" if m != "smsp__inst_executed.sum" else f"{vals.get(m, 0) / 1e6:9.1f}M"
            for m, _ in FULL_METRICS))
    return "\n".join(out), dict(traffic)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if args.launches:
        dst = os.path.join(PROF, f"{args.tag}_launches_{args.config}.csv")
        shutil.copy(args.launches, dst)
        with open(os.path.join(PROF, f"{args.tag}_launches_{args.config}_summary.txt"), "w") as f:
            f.write(launch_summary(args.launches) + "\n")
    if args.full:
        text, traffic = full_summary(args.full)
        with open(os.path.join(PROF, f"{args.tag}_ncu_full_{args.config}.txt"), "w") as f:
            f.write(f"ncu --set full --clock-control none --import-source on of bench.py --config {args.config} "
                    f"({os.path.basename(args.full)}); one launch each\n{args.note}\n{text}\n")
        with open(os.path.join(PROF, f"traffic_{args.config}.json"), "w") as f:
            json.dump({k: int(v) for k, v in traffic.items()} |
                      {"source": f"profiles/{args.tag}_ncu_full_{args.config}.txt",
                       "what": "dram__bytes_read.sum + dram__bytes_write.sum summed over the phase's "
                               "class launches (S, M, F), one step"}, f, indent=1)
    print(open(os.path.join(PROF, f"{args.tag}_launches_{args.config}_summary.txt")).read() if args.launches else "")


if __name__ == "__main__":
    main()
