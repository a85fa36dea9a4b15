"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle, bit-exact.

Corpus modelled on the reference's acceptance corpus (acceptance.cpp:61-153: sizes 1x1..64x64,
g in {1,2,4,8}, d in 0..1, both connectivities) plus multi-tile images that exercise the
cross-tile merge (tile = 32 x 256), ragged widths (scalar I/O path), batches, and the
structured nesting generator of config 3.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2006_09299_b200 import LabelingConfig
from tests.parity_util import compare_image

pytestmark = pytest.mark.gpu

SIZES = [(1, 1), (1, 7), (7, 1), (2, 2), (3, 5), (8, 8), (13, 9), (16, 16), (29, 23), (31, 33),
         (47, 61), (64, 64), (64, 1)]


def _check_batch(labeler, imgs, conn, where):
    cfg = LabelingConfig(connectivity=conn, relabel=True)
    res = labeler.label_batch(imgs, cfg)
    for i in range(imgs.shape[0]):
        ref = O.label_canonical(imgs[i], conn, want_labels=True)
        compare_image(res.image(i), ref, f"{where} #{i}")


@pytest.mark.parametrize("conn", [0, 1])
@pytest.mark.parametrize("w,h", SIZES)
def test_acceptance_corpus(labeler, conn, w, h):
    imgs = []
    for g in (1, 2, 4, 8):
        if g > min(w, h):
            continue
        for d in (0.0, 0.1, 0.3, 0.5, 0.7, 0.9, 1.0):
            for seed in (1, 2):
                imgs.append(O.generate(w, h, d, g, seed * 1000 + g))
    _check_batch(labeler, np.stack(imgs), conn, f"{w}x{h} conn{conn}")


@pytest.mark.parametrize("conn", [0, 1])
@pytest.mark.parametrize("w,h,d,g", [
    (300, 70, 0.5, 1), (300, 70, 0.45, 2), (513, 97, 0.5, 1), (257, 33, 0.6, 1),
    (256, 32, 0.5, 1), (512, 64, 0.55, 3), (1000, 333, 0.5, 2), (777, 129, 0.4, 1),
    (1024, 1024, 0.5, 1), (640, 480, 0.3, 4), (640, 480, 0.75, 1)])
def test_multi_tile(labeler, conn, w, h, d, g):
    img = O.generate(w, h, d, g, 7 + w + h)
    _check_batch(labeler, img[None], conn, f"{w}x{h} d{d} g{g}")


@pytest.mark.parametrize("conn", [0, 1])
@pytest.mark.parametrize("w,h,d,g", [
    (1000, 333, 0.5, 64), (777, 129, 0.3, 100), (2048, 256, 0.5, 256), (513, 97, 0.7, 40),
    (1030, 200, 0.05, 16), (900, 300, 0.8, 120), (256, 32, 1.0, 1), (300, 40, 0.0, 1)])
def test_flat_regions(labeler, conn, w, h, d, g):
    """Uniform tiles (one value over the whole tile: the single-component fast path of the
    analyze and emit passes) next to mixed ones, ragged edge tiles, flat holes filled."""
    img = O.generate(w, h, d, g, 11 + w + g)
    _check_batch(labeler, img[None], conn, f"{w}x{h} d{d} g{g}")


@pytest.mark.parametrize("conn", [0, 1])
def test_event_queue_rounds(labeler, conn):
    """Sparse-class tiles (<= 2048 runs) whose 4-row warps each hold ~254 essential union
    events -- rows [1010.., 1111.., 0101.., 0000..]: the all-1 row merges the singles above it,
    the all-0 row the background singles above it -- more than a warp's event queue (192):
    the shared drain must fall back to per-warp rounds (adjacent warps' queues would collide).
    One call of 640 tiles, so that the tiles go through the sparse class first (calls of at most
    one wave of dense-class CTAs go straight to the dense class)."""
    W, H = 2048, 320
    x = np.arange(W)
    imgs = []
    for bgval in (0, 1):
        for groups in [(4,), (4, 8, 40, 44), (0, 4, 8, 100, 104, 108), (24, 28, 60, 92, 124), (28, 32, 284)]:
            img = np.full((H, W), bgval, dtype=np.uint8)
            for r in groups:
                img[r] = (x % 2 == 0)
                img[r + 1] = 1
                img[r + 2] = (x % 2 == 1)
                img[r + 3] = 0
            imgs.append(img)
    _check_batch(labeler, np.stack(imgs[:8]), conn, "event rounds")


def test_batch_mixed(labeler):
    imgs = np.stack([O.generate(520, 96, d, g, 100 + i)
                     for i, (d, g) in enumerate([(0.1, 1), (0.5, 1), (0.9, 2), (0.5, 8), (0.0, 1), (1.0, 1)])])
    _check_batch(labeler, imgs, 0, "batch")


def test_nested_rings(labeler):
    img = O.generate_rings(512, 512, 64, 3, 0.02)
    _check_batch(labeler, img[None], 0, "rings")
    img = O.generate_rings(512, 512, 64, 5, 0.0)
    _check_batch(labeler, img[None], 0, "rings-clean")


def test_cfg2_cells(labeler):
    """A few full-size 2048^2 cells of BASELINE config 2."""
    imgs = np.stack([O.generate(2048, 2048, d, g, 1) for d, g in [(0.5, 1), (0.75, 1), (0.5, 4), (0.35, 16)]])
    res = labeler.label_batch(imgs, LabelingConfig())
    for i in range(imgs.shape[0]):
        ref = O.label_canonical(imgs[i], 0)
        compare_image(res.image(i), ref, f"cfg2 #{i}")


def _patterns(w, h):
    yy, xx = np.mgrid[0:h, 0:w]
    return {
        "checker": ((xx + yy) % 2).astype(np.uint8),          # one run per pixel: full-capacity path
        "vstripes": (xx % 2).astype(np.uint8),
        "hstripes": (yy % 2).astype(np.uint8),
        "dots": ((xx % 2 == 0) & (yy % 2 == 0)).astype(np.uint8),
        "diag": (((xx - yy) % 3) == 0).astype(np.uint8),
        "rings": (np.minimum(np.minimum(xx, yy), np.minimum(w - 1 - xx, h - 1 - yy)) % 2).astype(np.uint8),
    }


@pytest.mark.parametrize("conn", [0, 1])
def test_adversarial_patterns(labeler, conn):
    """Run-dense tiles (more runs than the fast tables hold) go through the full-capacity
    kernels; mixed batches exercise both paths in one call."""
    for (w, h) in [(256, 32), (300, 70), (1024, 96), (33, 17)]:
        pats = _patterns(w, h)
        imgs = np.stack(list(pats.values()) + [O.generate(w, h, 0.5, 1, 5)])
        _check_batch(labeler, imgs, conn, f"patterns {w}x{h}")


def test_error_contract(labeler):
    """labeling.hpp:271-273 and features.hpp:37-39: argument and overflow errors are raised
    before anything is allocated or launched."""
    from paper_2006_09299_b200 import LabelingConfig
    with pytest.raises(OverflowError):  # Sx = sum of columns could exceed int64
        labeler.label_device(0, 2**31 - 1, 2**31 - 1, 1, LabelingConfig(compute_features=True))
    with pytest.raises(ValueError):  # densify without relabel
        labeler.label_device(0, 64, 64, 1, LabelingConfig(relabel=False, densify_labels=True))
    with pytest.raises(ValueError):  # empty image
        labeler.label_device(0, 0, 64, 1, LabelingConfig())
    # the context stays usable
    img = O.generate(97, 65, 0.5, 1, 3)
    compare_image(labeler.label_batch(img[None], LabelingConfig(compute_features=True)).image(0),
                  O.label_canonical(img, 0), "after errors")


@pytest.mark.parametrize("seed", range(1, 13))
def test_structured_fuzz(labeler, seed):
    """Bands of adversarial row patterns (tools/fuzz_struct.py: checkerboards, stripes, merge rows
    under singles, diagonals, dots, noise, rectangles), in calls that go through the sparse class
    first and in small direct calls; the round-1 build failed its first batch (event-queue
    overflow), 2500 more batches (15 K images) ran clean on the current one."""
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_struct as F
    imgs, conn = F.batch(seed, big=seed % 3 != 0)
    _check_batch(labeler, imgs, conn, f"fuzz seed {seed}")


@pytest.mark.parametrize("seed", range(1, 19))
def test_shape_fuzz(labeler, seed):
    """Long thin structures across many seams and tile corners (tools/fuzz_shapes.py: spirals,
    serpentine combs, concentric rings, diagonal walks, corner pairs, mazes; alone, inverted,
    salted or XOR-ed), at sizes on and around the tile grid, with and without hole filling."""
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_shapes as F
    imgs, conn, relabel, fill = F.batch(seed)
    cfg = LabelingConfig(connectivity=conn, relabel=relabel, fill_holes=fill, compute_features=True,
                         compute_euler=True)
    res = labeler.label_batch(imgs, cfg)
    for i in range(imgs.shape[0]):
        ref = O.label_canonical(imgs[i], conn, want_labels=relabel)
        if relabel and fill:
            ref.labels = ref.top[ref.labels]
        compare_image(res.image(i), ref, f"shape fuzz seed {seed} #{i}")


@pytest.mark.parametrize("seed", [1, 2, 5])
def test_shape_fuzz_large(labeler, seed):
    """One 4-64 Mpixel shape image: structures spanning thousands of tiles (deep union chains
    over the seam graph, one component folding features from every tile)."""
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_shapes as F
    imgs, conn, relabel, fill = F.large(seed)
    cfg = LabelingConfig(connectivity=conn, relabel=relabel, fill_holes=fill, compute_features=True,
                         compute_euler=True)
    res = labeler.label_batch(imgs, cfg)
    ref = O.label_canonical(imgs[0], conn, want_labels=relabel)
    if relabel and fill:
        ref.labels = ref.top[ref.labels]
    compare_image(res.image(0), ref, f"large shape seed {seed} {imgs.shape}")


@pytest.mark.parametrize("seed", range(500000, 500008))
def test_shape_fuzz_densified_labels(labeler, seed):
    """Densified label images of shape-fuzz batches, with and without hole filling, against a
    flood fill of the (hole-filled) image (test_labeling.cpp:301-319)."""
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_shapes as F
    imgs, conn, _, fill = F.batch(seed)
    cfg = LabelingConfig(connectivity=conn, relabel=True, densify_labels=True, fill_holes=fill,
                         compute_features=True, compute_euler=True)
    res = labeler.label_batch(imgs, cfg)
    for i in range(imgs.shape[0]):
        _, comp, _ = O.flood_label(O.fill_holes(imgs[i], conn) if fill else imgs[i], conn)
        assert np.array_equal(res.labels[i].astype(np.int32), comp), f"seed {seed} #{i} fill={fill}"
