#!/usr/bin/env python
"""Small driver for ncu / per-cell timing: labels a device-generated batch and prints the
per-phase device times.

  python tools/prof_driver.py --cells 0.5:1,0.5:4 --copies 8 --iters 3
  python tools/prof_driver.py --sweep        # per-cell phase times over the config-2 sweep
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", default="0.5:1")
    ap.add_argument("--copies", type=int, default=8)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--size", type=int, default=2048)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--conn", type=int, default=0)
    ap.add_argument("--cfg2", action="store_true", help="the exact 105-image bench batch")
    args = ap.parse_args()

    import torch
    from paper_2006_09299_b200 import Connectivity, Labeler, LabelingConfig
    from paper_2006_09299_b200.runlab import cfg2_cells, generate_device

    lab = Labeler(0)
    lab.set_pipelines(1)  # phase events of one pipeline
    cfg = LabelingConfig(connectivity=Connectivity(args.conn), compute_features=True,
                         compute_euler=True, fill_holes=True)
    S = args.size

    def run(cells, copies, iters):
        B = len(cells) * copies
        imgs = torch.empty((B, S, S), dtype=torch.uint8, device="cuda")
        for i in range(B):
            d, g = cells[i % len(cells)]
            generate_device(imgs[i].data_ptr(), S, S, d, g, 1 if args.cfg2 else 1 + i // len(cells))
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            lab.label_device(imgs.data_ptr(), S, S, B, cfg)
            lab.sync()
            ts.append(lab.phase_times(0))
        t = ts[-1]
        return B, t

    if args.sweep:
        out = []
        for (d, g) in cfg2_cells():
            B, t = run([(d, g)], args.copies, 2)
            gpx = B * S * S / (t.total_ms / 1e3) / 1e9
            out.append({"d": d, "g": g, "analyze": t.analyze_ms / B, "merge": t.merge_ms / B,
                        "emit": t.emit_ms / B, "total": t.total_ms / B, "gpx": gpx})
            print(json.dumps(out[-1]), flush=True)
        return
    cells = [tuple(float(v) if i == 0 else int(v) for i, v in enumerate(c.split(":")))
             for c in args.cells.split(",")]
    if args.cfg2:
        cells = cfg2_cells()
        args.copies = 1
    B, t = run(cells, args.copies, args.iters)
    line = {"images": B, "analyze_ms": t.analyze_ms, "merge_ms": t.merge_ms, "emit_ms": t.emit_ms,
            "total_ms": t.total_ms, "gpx": B * S * S / (t.total_ms / 1e3) / 1e9}
    if os.environ.get("RUNLAB_GPU_KTIMES"):
        import ctypes as C
        from paper_2006_09299_b200 import _native as N
        L = N.load()
        L.rl_debug_launch_times.argtypes = [C.c_void_p, C.POINTER(C.c_float), C.c_int]
        ms = (C.c_float * 16)()
        n = L.rl_debug_launch_times(lab.ctx, ms, 16)
        names = ["analyze", "seams", "resolve", "scan", "cids", "tree", "emit"]
        line["launch_ms"] = {names[k] if k < len(names) else str(k): round(ms[k], 4) for k in range(n)}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
