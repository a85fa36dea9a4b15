#!/usr/bin/env python
"""One-off wide fuzz of the device path against the C oracle (beyond the test suite's 24 seeds):
random sizes (up to a few tiles each way), densities, granularities, connectivities, batch
sizes -- small calls (wide-call kernels) and batches padded past RUNLAB_GPU_WIDE_TILES (the
large-call kernels).  python tools/fuzz_many.py --seeds 400"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=200)
    ap.add_argument("--start", type=int, default=5000)
    args = ap.parse_args()
    import numpy as np
    from oracle import oracle as O
    from paper_2006_09299_b200 import Labeler, LabelingConfig
    from tests.parity_util import compare_image
    lab = Labeler(0)
    t0 = time.time()
    bad = 0
    for seed in range(args.start, args.start + args.seeds):
        rng = np.random.default_rng(seed)
        w = int(rng.choice([1, 5, 33, 256, 257, 600, 1000, 1537]))
        h = int(rng.choice([1, 2, 31, 33, 64, 97, 300, 513]))
        big = seed % 4 == 3  # enough images to exceed the wide-call threshold (large-call kernels)
        tiles = ((w + 255) // 256) * ((h + 31) // 32)
        n = int(min(64, max(1, 4200 // tiles + 1))) if big else int(rng.integers(1, 4))
        conn = int(rng.integers(0, 2))
        imgs = np.stack([O.generate(w, h, float(rng.random()), int(rng.integers(1, min(w, h, 8) + 1)),
                                    int(rng.integers(0, 1 << 30))) for _ in range(n)])
        cfg = LabelingConfig(connectivity=conn, compute_features=True, compute_euler=True, fill_holes=True,
                             relabel=True)
        res = lab.label_batch(imgs, cfg)
        for i in range(0, n, max(1, n // 4)):  # a sample of each batch
            want = O.label_canonical(imgs[i], conn, want_labels=True)
            want.labels = want.top[want.labels]
            try:
                compare_image(res.image(i), want, f"seed={seed} {w}x{h}x{n} conn={conn} image {i}")
            except AssertionError as e:
                bad += 1
                print("MISMATCH", e, flush=True)
    print(f"{args.seeds} seeds, {bad} mismatches, {time.time() - t0:.0f} s")
    lab.close()


if __name__ == "__main__":
    main()
