#!/usr/bin/env python
"""Phase times (one pipeline) of each rank's share of config 2 for N ranks: where the per-call
fixed cost of small shares goes.  python tools/shard_phases.py --world 8"""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--ranks", type=int, default=2)
    args = ap.parse_args()
    import torch
    from paper_2006_09299_b200 import Labeler, LabelingConfig
    from paper_2006_09299_b200.distributed import balanced_shards, image_cost
    from paper_2006_09299_b200.runlab import cfg2_cells, generate_device
    cells = cfg2_cells(); W = H = 2048
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    lab = Labeler(0); lab.set_pipelines(1)
    for r, idx in enumerate(balanced_shards([image_cost(d, g) for d, g in cells], args.world)[:args.ranks]):
        imgs = torch.empty((len(idx), H, W), dtype=torch.uint8, device="cuda")
        for j, i in enumerate(idx):
            generate_device(imgs[j].data_ptr(), W, H, cells[i][0], cells[i][1], 1)
        torch.cuda.synchronize()
        ts = []
        for k in range(8):
            lab.label_device(imgs.data_ptr(), W, H, len(idx), cfg); lab.sync()
            if k >= 3: ts.append(lab.phase_times(0))
        f = lambda a: round(sum(getattr(t, a) for t in ts) / len(ts), 4)
        print(json.dumps({"world": args.world, "rank": r, "images": len(idx), "analyze": f("analyze_ms"),
                          "merge": f("merge_ms"), "emit": f("emit_ms"), "total": f("total_ms")}))

if __name__ == "__main__":
    main()
