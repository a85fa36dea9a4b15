#!/usr/bin/env python
"""Shape-fuzz images (tools/fuzz_shapes.py) through the other entry points of the device path:

* strips: one image cut into 2-6 strips (in-process lockstep driver and the native
  multi-context rl_label_strips), every table / filled image / label image against the oracle;
* rl_label_into: a batch through host buffers in small chunks (compact record slots, escape
  lists, P4 staging of the filled image and of the input), both layouts of the post-fill
  features, against rl_label of the same batch (itself checked against the oracle);
* filter_components on the device over the first image's tree (random, hole, small-foreground and
  strided selections) against the oracle's restatement of the reference's filter;
* rl_fill_pbm: a P4 raster in, the hole-filled P4 raster out, against the oracle's filled image.

  python tools/fuzz_paths.py --seeds 300
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=100)
    ap.add_argument("--start", type=int, default=1)
    args = ap.parse_args()
    import torch
    import fuzz_shapes as F
    from oracle import oracle as O
    from paper_2006_09299_b200 import Labeler, LabelingConfig
    from tests.parity_util import compare_image
    from tests.test_gpu_into import _cap, _check, _into
    from tests.test_gpu_strips import _run, _run_native

    labs = [Labeler(0) for _ in range(6)]
    os.environ["RUNLAB_GPU_CHUNK_PX"] = str(1 << 19)
    try:
        small = Labeler(0)
    finally:
        del os.environ["RUNLAB_GPU_CHUNK_PX"]
    t0 = time.time()
    bad = 0

    def attempt(what, fn):
        nonlocal bad
        try:
            fn()
        except AssertionError as e:
            bad += 1
            print("MISMATCH", what, str(e)[:300], flush=True)

    for seed in range(args.start, args.start + args.seeds):
        if (seed - args.start) % 500 == 0 and seed != args.start:
            print(f"... {seed - args.start} done, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
        rng = np.random.default_rng(7_000_000 + seed)
        # --- strips
        W = int(rng.choice([255, 256, 257, 700, 1537, 2048, 2300]))
        H = int(rng.choice([64, 65, 97, 320, 333, 600, 1000]))
        img = F.image(rng, W, H)
        conn = int(rng.integers(0, 2))
        n = int(min(rng.integers(2, 7), (H + 31) // 32))
        cfg = LabelingConfig(connectivity=conn, compute_features=True, compute_euler=True, fill_holes=True,
                             relabel=True)
        want = O.label_canonical(img, conn, want_labels=True)
        want.labels = want.top[want.labels]
        dev = torch.from_numpy(img).cuda()

        def strips_case(native):
            got = (_run_native if native else _run)(labs, dev, W, H, n, cfg)
            compare_image(got, want, f"seed={seed} {W}x{H} conn={conn} strips={n} native={native}")
        attempt("strips", lambda: strips_case(False))
        if n >= 2:
            attempt("native strips", lambda: strips_case(True))

        # --- host-buffer path in small chunks
        w2, h2 = int(rng.choice([100, 256, 513, 1000])), int(rng.choice([33, 128, 300]))
        nb = int(rng.integers(2, 14))
        imgs = np.stack([F.image(rng, w2, h2) for _ in range(nb)])
        layout = int(rng.integers(0, 2))
        labels = bool(rng.integers(0, 2))
        cfg2 = LabelingConfig(connectivity=conn, compute_features=True, compute_euler=True, fill_holes=True,
                              relabel=labels)
        ref = small.label_batch(imgs, cfg2)

        def into_case():
            for i in range(0, nb, max(1, nb // 3)):
                w_i = O.label_canonical(imgs[i], conn, want_labels=labels)
                if labels:
                    w_i.labels = w_i.top[w_i.labels]
                compare_image(ref.image(i), w_i, f"seed={seed} batch image {i}")
            h_in = torch.from_numpy(imgs).pin_memory()
            o, outs = _into(small, h_in, cfg2, layout, _cap(ref), labels=labels)
            _check(o, outs, ref, layout, labels=labels)
        attempt(f"into seed={seed} {imgs.shape} layout={layout} labels={labels}", into_case)

        # --- filter_components on the device (analysis.hpp:89-125) over the first image's tree
        def filter_case():
            from paper_2006_09299_b200.runlab import filter_components
            comps = ref.image(0)["comps"]
            nc = comps.shape[0]
            ids = np.arange(nc)
            fg = (comps["flags"] & 1).astype(bool)
            sels = [(rng.random(nc) < float(rng.choice([0.05, 0.3, 0.7, 0.95]))) & (ids > 0),
                    (~fg) & (ids > 0), fg & (comps["s"] <= int(rng.integers(1, 40))),
                    (ids % int(rng.integers(2, 5)) == 0) & (ids > 0)]
            for k, sel in enumerate(sels):
                got = filter_components(comps, sel)
                want = O.filter_components(comps, sel)
                for j, (a, b) in enumerate(zip(got, want)):
                    assert a.tobytes() == b.tobytes(), f"selection {k} output {j} differs ({nc} components)"
        attempt(f"filter seed={seed} {imgs.shape}", filter_case)

        # --- PBM P4 raster in, hole-filled P4 raster out (`runlab fill`, tools/runlab.cpp:128-137)
        def pbm_case():
            from paper_2006_09299_b200.runlab import pack_p4
            im = imgs[int(rng.integers(0, nb))]
            hdr = f"P4\n{w2} {h2}\n".encode()
            got = small.fill_pbm(hdr + pack_p4(im).tobytes(), LabelingConfig(connectivity=conn, fill_holes=True))
            filled = O.label_canonical(im, conn).filled_image
            want = O.ref_write_pbm(filled) if O.ref_available() else hdr + pack_p4(filled).tobytes()
            assert got == want, "filled PBM differs"
        attempt(f"pbm seed={seed} {w2}x{h2} conn={conn}", pbm_case)
    print(f"{args.seeds} seeds, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
