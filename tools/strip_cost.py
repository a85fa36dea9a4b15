#!/usr/bin/env python
"""Cost model inputs of the strip path on one GPU: per-strip border components (the exchange
volume) and the phase times of one rank, for config 5 cut into N strips (in process)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--strips", type=int, default=8)
    ap.add_argument("--size", type=int, default=32768)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2006_09299_b200 import Labeler, LabelingConfig
    from paper_2006_09299_b200.runlab import generate_rows_device
    from paper_2006_09299_b200.strips import StripPhases, _maxima, strip_rows
    W = H = args.size
    rows = strip_rows(H, args.strips)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    bufs, phs = [], []
    for y0, h in rows:
        d = torch.empty((h, W), dtype=torch.uint8, device="cuda")
        generate_rows_device(d.data_ptr(), W, H, y0, h, 0.45, 4, 5)
        bufs.append(d)
        phs.append(StripPhases(Labeler(0)))
    torch.cuda.synchronize()
    for rep in range(2):
        t = {}
        t0 = time.perf_counter()
        infos = np.stack([ph.local(b.data_ptr(), W, H, y0, h, cfg) for ph, b, (y0, h) in zip(phs, bufs, rows)])
        torch.cuda.synchronize()
        t["local_all_ms"] = (time.perf_counter() - t0) * 1e3
        mn, mr = _maxima(infos)
        t0 = time.perf_counter()
        recs = [ph.export(mn, mr) for ph in phs]
        gathered = torch.cat(recs)
        torch.cuda.synchronize()
        t["export_ms"] = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        parts = phs[0].merge(gathered, infos, mn, mr)
        torch.cuda.synchronize()
        t["merge_one_rank_ms"] = (time.perf_counter() - t0) * 1e3
    print({"strips": args.strips, "nodes_per_strip": infos[:, 0].tolist(),
           "record_MB_per_strip": recs[0].numel() / 1e6, "gathered_MB": gathered.numel() / 1e6,
           "partials_k": int(parts[0].numel() // 3)} | t)


if __name__ == "__main__":
    main()
