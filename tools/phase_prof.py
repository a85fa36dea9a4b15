#!/usr/bin/env python
"""Per-phase latency of the analyze-pass tile CTAs (clock64 stamps of a profiling build).

Build here:  nvcc ... -DRL_PHASE_PROF -o paper_2006_09299_b200/librunlab_gpu_prof.so
Run on GPU:  python tools/phase_prof.py --cells 0.5:1 --copies 4
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RUNLAB_GPU_LIB", os.path.join(ROOT, "paper_2006_09299_b200", "librunlab_gpu_prof.so"))



def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", default="0.5:1")
    ap.add_argument("--copies", type=int, default=4)
    ap.add_argument("--cfg2", action="store_true", help="the cfg2 density/grain sweep, one image per cell")
    ap.add_argument("--size", type=int, default=2048)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2006_09299_b200 import Labeler, LabelingConfig, _native
    from paper_2006_09299_b200.runlab import cfg2_cells, generate_device

    L = _native.load()
    L.rl_debug_phase_buffer.argtypes = [C.c_void_p, C.c_int]
    cells = [tuple(float(v) if i == 0 else int(v) for i, v in enumerate(c.split(":"))) for c in args.cells.split(",")]
    if args.cfg2:
        cells, args.copies = list(cfg2_cells()), 1
    S = args.size
    B = len(cells) * args.copies
    imgs = torch.empty((B, S, S), dtype=torch.uint8, device="cuda")
    for i in range(B):
        d, g = cells[i % len(cells)]
        generate_device(imgs[i].data_ptr(), S, S, d, g, 1 + i)
    ntiles = B * (S // 32) * (S // 256)
    buf = torch.zeros(ntiles * 32, dtype=torch.int64, device="cuda")
    lab = Labeler(0)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    lab.label_device(imgs.data_ptr(), S, S, B, cfg)
    lab.sync()
    assert L.rl_debug_phase_buffer(C.c_void_p(buf.data_ptr()), ntiles) == 0
    buf.zero_()
    lab.label_device(imgs.data_ptr(), S, S, B, cfg)
    lab.sync()
    st = buf.view(ntiles, 32).cpu().numpy().astype(np.float64)
    # stamps in execution order (tile_ccl.cuh / kernels.cu RL_PHASE ids)
    seqs = {"analyze": [(0, "start"), (1, "load+init"), (2, "runs(scan)"), (13, "events (bit masks)"),
                        (14, "first contact+prefix"), (3, "pre-flatten"), (4, "union"), (5, "roots"),
                        (6, "border-mark"), (8, "scan/alloc"), (9, "map pass (walks)"),
                        (10, "border features+hdr"), (11, "perimeter"), (12, "nodes+cnt")],
            "emit": [(16, "prologue"), (18, "runs+prefix"), (19, "chunk init"), (20, "features"),
                     (21, "records+folds"), (22, "deferred folds"), (23, "flush"), (24, "filled image")]}
    for name, seq in seqs.items():
        ids = [k for k, _ in seq]
        ok = (st[:, ids] > 0).all(axis=1)
        if not ok.any():
            print(f"{name}: no tile with complete stamps")
            continue
        print(f"{name}: tiles with complete stamps: {ok.sum()} / {ntiles}; mean CTA latency "
              f"{(st[ok, ids[-1]] - st[ok, ids[0]]).mean():.0f} cycles (chunk phases: last chunk)")
        for (a, _), (b, label) in zip(seq, seq[1:]):
            d = st[ok, b] - st[ok, a]
            print(f"  {label:24s} {d.mean():9.0f} cycles  (p90 {np.percentile(d, 90):9.0f})")


if __name__ == "__main__":
    main()
