#!/usr/bin/env python
"""Projected batch scaling of config 2 on one GPU: for N = 1, 2, 4, 8 ranks, every rank's share
of the 105 images (the bench's cost-balanced sharding, distributed.balanced_shards) is timed
alone with CUDA events; the projected N-GPU step is the slowest rank's time (no collective is on
the data path: images are independent).  Writes one JSON line.

  python tools/scale_projection.py [--steps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_2006_09299_b200 import Labeler, LabelingConfig
    from paper_2006_09299_b200.distributed import balanced_shards, image_cost
    from paper_2006_09299_b200.runlab import cfg2_cells, generate_device
    cells = cfg2_cells()
    W = H = 2048
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    lab = Labeler(0)
    st = torch.cuda.ExternalStream(lab.stream())
    out = {"workload": "cfg2: 105 x 2048^2", "method": "each rank's shard timed alone on one B200; step = max over ranks",
           "ranks": {}}
    base = None
    for world in (1, 2, 4, 8):
        per = []
        for idx in balanced_shards([image_cost(d, g) for d, g in cells], world):
            imgs = torch.empty((len(idx), H, W), dtype=torch.uint8, device="cuda")
            for j, i in enumerate(idx):
                generate_device(imgs[j].data_ptr(), W, H, cells[i][0], cells[i][1], 1)
            torch.cuda.synchronize()
            for _ in range(4):
                lab.label_device(imgs.data_ptr(), W, H, len(idx), cfg)
                lab.sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.steps):
                lab.label_device(imgs.data_ptr(), W, H, len(idx), cfg)
            e1.record(st)
            torch.cuda.synchronize()
            lab.sync()
            per.append(e0.elapsed_time(e1) / args.steps)
            del imgs
        step = max(per)
        gpx = len(cells) * W * H / step / 1e6
        base = base or gpx
        out["ranks"][str(world)] = {"rank_ms": [round(t, 4) for t in per], "step_ms": round(step, 4),
                                    "gpx": round(gpx, 1), "efficiency": round(gpx / (base * world), 3)}
    lab.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
