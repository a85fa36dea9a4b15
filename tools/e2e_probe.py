#!/usr/bin/env python
"""Time rl_label_into on config 2 under host-path variants (env knobs read at context creation).

  python tools/e2e_probe.py --variants "base;RUNLAB_GPU_NO_PACKED_RECORDS=1;RUNLAB_GPU_HOST_THREADS=8"
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="base")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--spin", action="store_true", help="keep one SM busy on a side stream (power-state probe)")
    args = ap.parse_args()
    import torch
    from paper_2006_09299_b200 import Labeler, LabelingConfig, _native as N
    from paper_2006_09299_b200.runlab import cfg2_cells, generate_device, pack_p4
    cells = list(cfg2_cells())
    B, S = len(cells), 2048
    imgs = torch.empty((B, S, S), dtype=torch.uint8, device="cuda")
    for i, (d, g) in enumerate(cells):
        generate_device(imgs[i].data_ptr(), S, S, d, g, 1)
    torch.cuda.synchronize()
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    h_in = imgs.cpu().pin_memory()
    h_p4 = torch.from_numpy(pack_p4(h_in.numpy())).pin_memory()
    h_fill = torch.empty_like(h_in).pin_memory()
    h_fp4 = torch.empty_like(h_p4).pin_memory()
    cap = 12_000_000
    h_comps = torch.empty(cap * 48, dtype=torch.uint8, pin_memory=True)
    h_top = torch.empty(cap * 4, dtype=torch.uint8, pin_memory=True)
    h_filled = torch.empty(cap * 40, dtype=torch.uint8, pin_memory=True)
    h_summ = torch.empty(B * 5, dtype=torch.int64, pin_memory=True)
    h_off = torch.empty(B + 1, dtype=torch.int64, pin_memory=True)
    for var in args.variants.split(";"):
        env = {} if var == "base" else dict(kv.split("=") for kv in var.split(","))
        outsel = env.pop("OUT", "fill+comps")  # which outputs: fill, comps, or both
        os.environ.update(env)
        lab = Labeler(0)
        for k in env:
            del os.environ[k]
        for fmt, src, dst in ((N.RL_PIXELS_U8, h_in, h_fill), (N.RL_PIXELS_P4, h_p4, h_fp4)):
            wf, wc = "fill" in outsel, "comps" in outsel
            outs = N.RlHostOutputs(dst.data_ptr() if wf else None, None, h_comps.data_ptr() if wc else None,
                                   h_top.data_ptr() if wc else None, h_filled.data_ptr() if wc else None,
                                   cap, h_summ.data_ptr(), h_off.data_ptr(), 0, 0, 0, 1, 0)
            lab.label_into(src.data_ptr(), S, S, B, cfg, outs, pixel_format=fmt)
            ts = []
            side = torch.cuda.Stream()
            for _ in range(args.steps):
                if args.spin:
                    with torch.cuda.stream(side):
                        torch.cuda._sleep(2_000_000_00 // 10)  # ~10 ms at 2 GHz
                t0 = time.perf_counter()
                lab.label_into(src.data_ptr(), S, S, B, cfg, outs, pixel_format=fmt)
                ts.append(time.perf_counter() - t0)
            ts.sort()
            print(f"{var:45s} {'u8' if fmt == N.RL_PIXELS_U8 else 'p4'}  min {ts[0]*1e3:6.2f} ms  "
                  f"med {ts[len(ts)//2]*1e3:6.2f} ms  d2h {outs.d2h_bytes/1e6:6.1f} MB  "
                  f"{B*S*S/ts[len(ts)//2]/1e9:6.1f} Gpx/s", flush=True)
        lab.close()
    # raw D2H bandwidth in this process afterwards (is something in the process throttling PCIe?)
    N = 24 << 20
    dbuf = torch.empty(N, dtype=torch.uint8, device="cuda")
    hb = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    cs = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    with torch.cuda.stream(cs):
        for _ in range(20):
            hb.copy_(dbuf, non_blocking=True)
    e1.record(cs)
    torch.cuda.synchronize()
    print(f"raw D2H in-process: {20 * N / e0.elapsed_time(e1) / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
