#!/usr/bin/env python
"""Structured fuzz of the device path against the C oracle: images built from bands of rows
with adversarial patterns (checkerboards, stripes, merge rows under singles, diagonals, uniform
bands, noise at any density/grain, random rectangles), so that tiles land on every capacity
edge -- event-queue rounds, component/border-component limits of each class, emit feature
chunks, fold-table overflow -- in calls large enough to go through the sparse class first
(> one wave of dense-class CTAs) and in small direct calls.

  python tools/fuzz_struct.py --batches 60
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def band(rng, rows: int, w: int) -> np.ndarray:
    """One band of `rows` rows with a random pattern."""
    x = np.arange(w)
    y = np.arange(rows)[:, None]
    k = int(rng.integers(0, 10))
    ph = int(rng.integers(0, 2))
    if k == 0:
        return np.full((rows, w), ph, np.uint8)
    if k == 1:  # checkerboard
        return ((x[None, :] + y + ph) & 1).astype(np.uint8)
    if k == 2:  # vertical stripes of period p
        p = int(rng.integers(2, 9))
        return np.broadcast_to(((x // max(1, p // 2)) + ph) & 1, (rows, w)).astype(np.uint8)
    if k == 3:  # singles / merge row / singles / merge row (many essential union events)
        out = np.empty((rows, w), np.uint8)
        for r in range(rows):
            q = (r + ph) & 3
            out[r] = (x % 2 == 0) if q == 0 else 1 if q == 1 else (x % 2 == 1) if q == 2 else 0
        return out
    if k == 4:  # diagonals of period p
        p = int(rng.integers(2, 7))
        return (((x[None, :] + (1 if ph else -1) * y) % p) == 0).astype(np.uint8)
    if k == 5:  # horizontal stripes
        return np.broadcast_to(((y // int(rng.integers(1, 4))) + ph) & 1, (rows, w)).astype(np.uint8)
    if k in (6, 7):  # noise at a random density and grain
        d = float(rng.random())
        g = int(rng.choice([1, 1, 2, 3, 4, 8]))
        blocks = rng.random(((rows + g - 1) // g, (w + g - 1) // g)) < d
        return np.kron(blocks, np.ones((g, g), bool))[:rows, :w].astype(np.uint8)
    if k == 8:  # dots (one isolated pixel per 2x2): many components
        return (((x[None, :] % 2) == ph) & ((y % 2) == 0)).astype(np.uint8)
    # random rectangles on a uniform ground (holes, nesting)
    out = np.full((rows, w), ph, np.uint8)
    for _ in range(int(rng.integers(1, 40))):
        r0, c0 = int(rng.integers(0, rows)), int(rng.integers(0, w))
        out[r0:r0 + int(rng.integers(1, 40)), c0:c0 + int(rng.integers(1, 300))] ^= 1
    return out


def image(rng, w: int, h: int) -> np.ndarray:
    img = np.empty((h, w), np.uint8)
    r = 0
    while r < h:
        n = int(rng.choice([1, 2, 3, 4, 5, 8, 12, 16, 32, 64]))
        n = min(n, h - r)
        img[r:r + n] = band(rng, n, w)
        r += n
    return img


def batch(seed: int, big: bool):
    """(images, connectivity): big calls exceed one wave of dense-class CTAs."""
    rng = np.random.default_rng(seed)
    if big:
        w, h, n = int(rng.choice([2048, 2000, 1537])), int(rng.choice([320, 333, 290])), 8
    else:
        w, h, n = int(rng.choice([256, 600, 1000, 1537])), int(rng.choice([32, 97, 300])), int(rng.integers(1, 4))
    return np.stack([image(rng, w, h) for _ in range(n)]), int(rng.integers(0, 2))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=40)
    ap.add_argument("--start", type=int, default=1)
    args = ap.parse_args()
    from oracle import oracle as O
    from paper_2006_09299_b200 import Labeler, LabelingConfig
    from tests.parity_util import compare_image
    lab = Labeler(0)
    t0 = time.time()
    bad = n_img = 0
    for seed in range(args.start, args.start + args.batches):
        if (seed - args.start) % 500 == 0 and seed != args.start:
            print(f"... {seed - args.start} done, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
        imgs, conn = batch(seed, big=seed % 3 != 0)
        cfg = LabelingConfig(connectivity=conn, relabel=True)
        res = lab.label_batch(imgs, cfg)
        for i in range(imgs.shape[0]):
            n_img += 1
            try:
                compare_image(res.image(i), O.label_canonical(imgs[i], conn, want_labels=True),
                              f"seed={seed} {imgs.shape} conn={conn} image {i}")
            except AssertionError as e:
                bad += 1
                print("MISMATCH", e, flush=True)
    print(f"{args.batches} batches, {n_img} images, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
    lab.close()


if __name__ == "__main__":
    main()
