#!/usr/bin/env python
"""The reference's benchmark sweep (bench.hpp:20-207, `runlab bench`) on the GPU.

For each density x granularity cell, `--seeds` images (seeds base_seed .. base_seed+seeds-1,
the reference's BenchSpec) are labeled as one device-resident batch per configuration variant
(bench.hpp:96-121: base / euler / fill / features / relabel), `--warmup` untimed then
`--iterations` timed calls (CUDA events).  Output: the reference's CSV schema
(d,g,config,step,min_ns_px,med_ns_px,max_ns_px,min_cpp,med_cpp,max_cpp) with steps `total`,
`analyze`, `merge`, `emit` (the device phases; the reference's are encode/unify/closure/relabel).
ns_px = batch time / (seeds * w * h); cpp columns with --clock-ghz.

  python tools/bench_sweep.py --densities 0:1:0.05 --granularities 1,2,4,8,16 > sweep.csv
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse_densities(text: str) -> list[float]:
    """'start:stop:step' (inclusive) or 'a,b,c' (tools/runlab.cpp:35-55)."""
    if ":" in text:
        a, b, s = (float(v) for v in text.split(":"))
        if s <= 0:
            raise SystemExit("--densities: expected start:stop:step")
        out, k = [], 0
        while a + k * s <= b + 1e-9:
            out.append(min(round(a + k * s, 12), 1.0))
            k += 1
    else:
        out = [float(v) for v in text.split(",")]
    if any(d < 0 or d > 1 for d in out):
        raise SystemExit("--densities: values must be in [0, 1]")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=2048)
    ap.add_argument("--height", type=int, default=2048)
    ap.add_argument("--densities", default="0:1:0.05")
    ap.add_argument("--granularities", default="1,2,4,8,16")
    ap.add_argument("--seeds", type=int, default=5)
    ap.add_argument("--base-seed", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--iterations", type=int, default=3)
    ap.add_argument("--clock-ghz", type=float, default=0.0)
    ap.add_argument("--connectivity", choices=["fg8bg4", "fg4bg8"], default="fg8bg4")
    args = ap.parse_args()

    import torch
    from paper_2006_09299_b200 import Connectivity, Labeler, LabelingConfig
    from paper_2006_09299_b200.runlab import generate_device

    conn = Connectivity(0 if args.connectivity == "fg8bg4" else 1)
    variants = [("base", LabelingConfig(connectivity=conn)),
                ("euler", LabelingConfig(connectivity=conn, compute_euler=True)),
                ("fill", LabelingConfig(connectivity=conn, fill_holes=True)),
                ("features", LabelingConfig(connectivity=conn, compute_features=True)),
                ("relabel", LabelingConfig(connectivity=conn, relabel=True))]
    W, H, S = args.width, args.height, args.seeds
    px = W * H * S
    lab = Labeler(0)
    imgs = torch.empty((S, H, W), dtype=torch.uint8, device="cuda")

    def num(v):
        return f"{v:.6g}"

    print("d,g,config,step,min_ns_px,med_ns_px,max_ns_px,min_cpp,med_cpp,max_cpp")
    for d in parse_densities(args.densities):
        for g in (int(v) for v in args.granularities.split(",")):
            for s in range(S):
                generate_device(imgs[s].data_ptr(), W, H, d, g, args.base_seed + s)
            torch.cuda.synchronize()
            for name, cfg in variants:
                for _ in range(args.warmup):
                    lab.label_device(imgs.data_ptr(), W, H, S, cfg)
                    lab.sync()
                ts = []
                for _ in range(args.iterations):
                    lab.label_device(imgs.data_ptr(), W, H, S, cfg)
                    lab.sync()
                    ts.append(lab.phase_times(0))
                for step, vals in (("total", [t.total_ms for t in ts]), ("analyze", [t.analyze_ms for t in ts]),
                                   ("merge", [t.merge_ms for t in ts]), ("emit", [t.emit_ms for t in ts])):
                    ns = sorted(v * 1e6 / px for v in vals)
                    row = [num(d), str(g), name, step, num(ns[0]), num(statistics.median(ns)), num(ns[-1])]
                    row += [num(v * args.clock_ghz) for v in (ns[0], statistics.median(ns), ns[-1])] \
                        if args.clock_ghz > 0 else ["", "", ""]
                    print(",".join(row), flush=True)


if __name__ == "__main__":
    main()
