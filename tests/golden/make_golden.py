#!/usr/bin/env python
"""Regenerate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libref_runlab.so,
compiled from the unmodified headers under /root/reference by oracle/Makefile).

Run in a container that has /root/reference:  make -C oracle && python tests/golden/make_golden.py

Fixtures (canonical form: components numbered by raster order of first pixel, exterior 0):
  fig_example.npz    the 15x7 grid of the paper's Fig. 3 (proj/tests/helpers.hpp:25-35)
  ring_hole_dot.npz  7x7 nesting chain (proj/tests/helpers.hpp:38-48)
  two_dots.npz       "two dots, one with a hole" (proj/tests/test_analysis.cpp:130-144)
  random_*.npz       seeded generate() images, both connectivities
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def grid(rows):
    return np.array([[1 if ch == "1" else 0 for ch in r] for r in rows], dtype=np.uint8)


FIG_EXAMPLE = grid([
    "011111111111110",
    "010000010000010",
    "010111010111010",
    "010101000101010",
    "010101111101010",
    "010100000001000",
    "011111111111110",
])
RING_HOLE_DOT = grid([
    "0000000",
    "0111110",
    "0100010",
    "0101010",
    "0100010",
    "0111110",
    "0000000",
])
TWO_DOTS = grid([
    "000111000",
    "010101000",
    "000111000",
])

RANDOM_SPECS = [  # (w, h, density, granularity, seed)
    (29, 23, 0.5, 1, 21), (33, 21, 0.45, 1, 31), (25, 25, 0.55, 1, 51), (64, 64, 0.5, 2, 7),
    (57, 1, 0.5, 1, 3), (1, 40, 0.5, 1, 4), (300, 70, 0.5, 1, 11), (300, 70, 0.6, 4, 12),
]


def dump(name: str, img: np.ndarray, conn: int) -> None:
    r = O.ref_label_canonical(img, conn, want_labels=True)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"), image=img, conn=conn, n_components=r.n_components,
        n_fg=r.n_fg, n_holes=r.n_holes, euler=r.euler, n_survivors=r.n_survivors, comps=r.comps,
        top=r.top, filled=r.filled, filled_image=r.filled_image, labels=r.labels)
    print(f"{name}: C_pre={r.n_components} C_post={r.n_survivors} euler={r.euler}")


def main() -> None:
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libref_runlab.so missing: run `make -C oracle` where "
                         "/root/reference exists")
    dump("fig_example", FIG_EXAMPLE, 0)
    dump("ring_hole_dot", RING_HOLE_DOT, 0)
    dump("two_dots", TWO_DOTS, 0)
    for (w, h, d, g, s) in RANDOM_SPECS:
        for conn in (0, 1):
            img = O.generate(w, h, d, g, s)
            dump(f"random_{w}x{h}_d{int(d * 100)}_g{g}_s{s}_c{conn}", img, conn)


if __name__ == "__main__":
    main()
