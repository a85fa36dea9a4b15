#!/usr/bin/env python
"""rl_label_into timeline of one large image (config 5 by default): RUNLAB_GPU_DEBUG_TIMELINE=1
prints the per-chunk copy/kernel/host stamps.  python tools/e2e_one.py [--size 32768]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=32768)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    import torch
    from paper_2006_09299_b200 import Labeler, LabelingConfig, _native as N
    from paper_2006_09299_b200.runlab import generate_device
    S = args.size
    img = torch.empty((S, S), dtype=torch.uint8, device="cuda")
    generate_device(img.data_ptr(), S, S, 0.45, 4, 5)
    h_in = img.cpu().pin_memory()
    h_fill = torch.empty_like(h_in).pin_memory()
    cap = 8_000_000
    h_comps = torch.empty(cap * 48, dtype=torch.uint8, pin_memory=True)
    h_top = torch.empty(cap * 4, dtype=torch.uint8, pin_memory=True)
    h_filled = torch.empty(cap * 40, dtype=torch.uint8, pin_memory=True)
    h_summ = torch.empty(5, dtype=torch.int64, pin_memory=True)
    h_off = torch.empty(2, dtype=torch.int64, pin_memory=True)
    lab = Labeler(0)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    outs = N.RlHostOutputs(h_fill.data_ptr(), None, h_comps.data_ptr(), h_top.data_ptr(), h_filled.data_ptr(), cap,
                           h_summ.data_ptr(), h_off.data_ptr(), 0, 0, 0, 1, 0)
    for i in range(args.steps):
        t0 = time.perf_counter()
        lab.label_into(h_in.data_ptr(), S, S, 1, cfg, outs)
        print(f"step {i}: {(time.perf_counter() - t0) * 1e3:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
