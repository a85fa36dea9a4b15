#!/usr/bin/env python
"""Shape fuzz of the device path against the C oracle: long thin structures that cross many
tile seams and corners -- spirals, serpentine combs, concentric rings (deep inclusion trees),
random walks, diagonal pairs pinned on tile corners, lattices with one defect per cell -- alone,
inverted, or XOR-ed with noise, at sizes on and around the tile grid (32-row x 256-column
tiles) from 1 pixel to a few thousand columns, in small direct calls and in batches large
enough for the sparse-class-first kernels.  Complements tools/fuzz_many.py (noise) and
tools/fuzz_struct.py (row bands).

  python tools/fuzz_shapes.py --batches 200
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TH, TW = 32, 256


def spiral(rng, w: int, h: int) -> np.ndarray:
    """Rectangular spiral: arm `a` pixels wide, gap `b`: one long snake and one long channel."""
    a, b = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    img = np.zeros((h, w), np.uint8)
    x0, y0, x1, y1 = 0, 0, w, h
    p = a + b
    while x1 - x0 > 0 and y1 - y0 > 0:
        img[y0:min(y0 + a, y1), x0:x1] = 1                       # top
        img[y0:y1, max(x1 - a, x0):x1] = 1                       # right
        img[max(y1 - a, y0):y1, x0:x1] = 1                       # bottom
        img[min(y0 + p, y1):y1, x0:min(x0 + a, x1)] = 1          # left, open at the top: the way in
        if y0 + p < y1:
            img[y0 + a:y0 + p, x0:min(x0 + a, x1)] = 0
            img[y0 + p:min(y0 + p + a, y1), x0:min(x0 + p, x1)] = 1  # link to the next ring
        x0, y0, x1, y1 = x0 + p, y0 + p, x1 - p, y1 - p
    return img


def comb(rng, w: int, h: int) -> np.ndarray:
    """Serpentine: teeth of period p joined alternately at the top and the bottom of each band."""
    p = int(rng.integers(1, 4))
    bh = int(rng.choice([3, 5, 8, 17, 31, 32, 33, 64, 100]))
    vertical = bool(rng.integers(0, 2))
    W, H = (w, h) if vertical else (h, w)
    x = np.arange(W)
    img = np.zeros((H, W), np.uint8)
    tooth = ((x // p) % 2 == 0)
    for r0 in range(0, H, bh):
        r1 = min(r0 + bh, H)
        img[r0:r1] = tooth
        k = (x // p) // 2
        if r1 - r0 >= 2:
            img[r0] |= ((k % 2 == 0) & ((x // p) % 2 == 1)).astype(np.uint8)      # joins at the top
            img[r1 - 1] |= ((k % 2 == 1) & ((x // p) % 2 == 1)).astype(np.uint8)  # joins at the bottom
    return img if vertical else np.ascontiguousarray(img.T)


def rings(rng, w: int, h: int) -> np.ndarray:
    """Concentric square or diamond rings of random widths around random centres (XOR-ed)."""
    yy, xx = np.mgrid[0:h, 0:w]
    img = np.zeros((h, w), np.uint8)
    for _ in range(int(rng.integers(1, 4))):
        cx, cy = int(rng.integers(0, w)), int(rng.integers(0, h))
        d = np.maximum(abs(xx - cx), abs(yy - cy)) if rng.integers(0, 2) else abs(xx - cx) + abs(yy - cy)
        widths = rng.integers(1, 4, size=64)
        edges = np.cumsum(widths)
        ring = np.searchsorted(edges, d % int(edges[-1]), side="right")
        img ^= (ring & 1).astype(np.uint8)
    return img


def walks(rng, w: int, h: int) -> np.ndarray:
    """Thin random walks with diagonal steps (8- vs 4-connectivity differs on every step)."""
    img = np.zeros((h, w), np.uint8)
    for _ in range(int(rng.integers(1, 30))):
        x, y = int(rng.integers(0, w)), int(rng.integers(0, h))
        n = int(rng.integers(10, 4 * (w + h)))
        dx = rng.integers(-1, 2, size=n)
        dy = rng.integers(-1, 2, size=n)
        bias = int(rng.integers(0, 4))
        if bias == 1: dx[:] = 1
        if bias == 2: dy[:] = 1
        if bias == 3: dx[:], dy[:] = 1, np.where(rng.random(n) < 0.5, 1, -1)
        xs = np.clip(x + np.cumsum(dx), 0, w - 1)
        ys = np.clip(y + np.cumsum(dy), 0, h - 1)
        img[ys, xs] = 1
    return img


def corners(rng, w: int, h: int) -> np.ndarray:
    """Diagonal pairs and small crosses on tile corners and seams, elsewhere empty or sparse."""
    img = (rng.random((h, w)) < float(rng.choice([0.0, 0.0, 0.01, 0.2]))).astype(np.uint8)
    for ty in range(0, h + TH, TH):
        for tx in range(0, w + TW, TW):
            k = int(rng.integers(0, 6))
            pts = {0: [(-1, -1), (0, 0)], 1: [(-1, 0), (0, -1)], 2: [(-1, -1), (0, 0), (-1, 0)],
                   3: [(-1, -1), (0, 0), (-1, 0), (0, -1)], 4: [(-2, -2), (-1, -1), (0, 0), (1, 1)],
                   5: [(-2, 1), (-1, 0), (0, -1), (1, -2)]}[k]
            for dy, dx in pts:
                y, x = ty + dy, tx + dx
                if 0 <= y < h and 0 <= x < w:
                    img[y, x] = 1
            # clear the other pixels of the 2x2 around the corner so the pair is the only link
            if k in (0, 1):
                for dy, dx in [(-1, -1), (0, 0), (-1, 0), (0, -1)]:
                    y, x = ty + dy, tx + dx
                    if (dy, dx) not in pts and 0 <= y < h and 0 <= x < w:
                        img[y, x] = 0
    return img


def lattice(rng, w: int, h: int) -> np.ndarray:
    """Grid lines of period p with one gap per cell wall at random: mazes (many unions, few comps)."""
    p = int(rng.integers(2, 9))
    yy, xx = np.mgrid[0:h, 0:w]
    img = ((xx % p == 0) | (yy % p == 0)).astype(np.uint8)
    holes = rng.random((h, w)) < 1.0 / p
    img[holes & (img == 1) & ~((xx % p == 0) & (yy % p == 0))] = 0
    return img


FAMILIES = [spiral, comb, rings, walks, corners, lattice]


def dims(rng, big: bool):
    def around(step, lo, hi):
        base = int(rng.integers(lo, hi + 1)) * step
        return max(1, base + int(rng.choice([-1, 0, 0, 1, int(rng.integers(-step + 1, step))])))
    if big:
        return around(TW, 4, 10), around(TH, 8, 14)
    k = int(rng.integers(0, 5))
    if k == 0: return int(rng.integers(1, 9)), around(TH, 1, 40)         # a sliver, tall
    if k == 1: return around(TW, 4, 16), int(rng.integers(1, 9))         # a sliver, wide
    if k == 2: return around(TW, 1, 1), around(TH, 1, 30)                # one tile column
    return around(TW, 1, 5), around(TH, 1, 12)


def image(rng, w: int, h: int) -> np.ndarray:
    img = FAMILIES[int(rng.integers(0, len(FAMILIES)))](rng, w, h)
    m = int(rng.integers(0, 6))
    if m == 1:
        img = 1 - img
    elif m == 2:  # salt
        img = img ^ (rng.random((h, w)) < float(rng.choice([0.002, 0.02, 0.1]))).astype(np.uint8)
    elif m == 3:  # a second family over it
        img = img ^ FAMILIES[int(rng.integers(0, len(FAMILIES)))](rng, w, h)
    elif m == 4:  # bands of two families
        other = FAMILIES[int(rng.integers(0, len(FAMILIES)))](rng, w, h)
        cut = int(rng.integers(0, h + 1))
        img = np.concatenate([img[:cut], other[cut:]])
    return np.ascontiguousarray(img.astype(np.uint8))


def large(seed: int):
    """One image of 4-64 Mpixel: structures spanning thousands of tiles (union chains across the
    whole seam graph, one component folding features from every tile)."""
    rng = np.random.default_rng(1_000_000 + seed)
    w = int(rng.choice([2048, 4096, 4097, 5000, 8192])) + int(rng.choice([0, 0, -1, 1, 37]))
    h = int(rng.choice([2048, 3000, 4096, 8192])) + int(rng.choice([0, 0, -1, 1, 13]))
    return image(rng, w, h)[None], int(rng.integers(0, 2)), bool(rng.integers(0, 2)), bool(rng.integers(0, 2))


def batch(seed: int):
    rng = np.random.default_rng(seed)
    big = seed % 3 == 0
    w, h = dims(rng, big)
    n = int(rng.integers(6, 10)) if big else int(rng.integers(1, 4))
    return (np.stack([image(rng, w, h) for _ in range(n)]), int(rng.integers(0, 2)), bool(rng.integers(0, 4)),
            bool(rng.integers(0, 2)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=60)
    ap.add_argument("--start", type=int, default=1)
    ap.add_argument("--large", action="store_true", help="one 4-64 Mpixel image per seed")
    ap.add_argument("--ref", action="store_true",
                    help="check against the reference itself (oracle/_ref) instead of the C restatement")
    ap.add_argument("--densify", action="store_true",
                    help="densified label images against a flood fill of the (hole-filled) image "
                         "(test_labeling.cpp:301-319) instead of the canonical tables")
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
        imgs, conn, relabel, fill = (large if args.large else batch)(seed)
        if args.densify:
            cfg = LabelingConfig(connectivity=conn, relabel=True, densify_labels=True, fill_holes=fill,
                                 compute_features=True, compute_euler=True)
            res = lab.label_batch(imgs, cfg)
            for i in range(imgs.shape[0]):
                n_img += 1
                _, comp, _ = O.flood_label(O.fill_holes(imgs[i], conn) if fill else imgs[i], conn)
                if not np.array_equal(res.labels[i].astype(np.int32), comp):
                    bad += 1
                    print(f"MISMATCH seed={seed} {imgs.shape} conn={conn} fill={fill} image {i}: densified labels "
                          f"differ at {int((res.labels[i].astype(np.int32) != comp).sum())} pixels", flush=True)
            continue
        cfg = LabelingConfig(connectivity=conn, relabel=relabel, fill_holes=fill, compute_features=True,
                             compute_euler=True)
        res = lab.label_batch(imgs, cfg)
        for i in range(imgs.shape[0]):
            n_img += 1
            try:
                want = (O.ref_label_canonical if args.ref else O.label_canonical)(imgs[i], conn, want_labels=relabel)
                if relabel and fill:  # the label image of a hole-filling call carries post-fill roots
                    want.labels = want.top[want.labels]
                compare_image(res.image(i), want, f"seed={seed} {imgs.shape} conn={conn} fill={fill} image {i}")
            except AssertionError as e:
                bad += 1
                print("MISMATCH", e, flush=True)
    print(f"{args.batches} batches, {n_img} images, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
    lab.close()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
