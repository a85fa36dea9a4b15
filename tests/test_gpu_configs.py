"""GPU parity at BASELINE.json's full configuration sizes.

cfg1 (1024^2), cfg3 (4096^2 nested rings) and a sample of cfg4 (1920x1080) are compared with the
oracle bit-exactly.  cfg5 (one 32768^2 image, 1 Gpixel) is compared bit-exactly as well (the C
oracle needs ~20 s for it) plus size-independent invariants: the pixel mass of all components
sums to P, the Euler number equals the bit-quad count, every parent id is smaller than its child.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from paper_2006_09299_b200 import LabelingConfig
from tests.parity_util import compare_image

pytestmark = pytest.mark.gpu


def _invariants(got: dict, img: np.ndarray, conn: int = 0):
    h, w = img.shape
    comps = got["comps"]
    assert int(comps["s"].sum()) == w * h
    assert got["euler"] == O.bitquad_euler(img, conn)
    ids = np.arange(comps.shape[0], dtype=np.uint32)
    assert np.all(comps["parent"][1:] < ids[1:])
    assert np.all(got["top"] <= ids)
    # parities alternate along the tree (test_labeling.cpp:273-279)
    par = comps["parent"][1:].astype(np.int64)
    assert np.all((comps["flags"][1:] & 1) != (comps["flags"][par] & 1))


def test_cfg1_full(labeler):
    img = O.generate(1024, 1024, 0.5, 1, 1)
    res = labeler.label_batch(img[None], LabelingConfig(relabel=True))
    compare_image(res.image(0), O.label_canonical(img, 0, want_labels=True), "cfg1")
    _invariants(res.image(0), img)


def test_cfg3_full(labeler):
    img = O.generate_rings(4096, 4096, 64, 3, 0.02)
    res = labeler.label_batch(img[None], LabelingConfig())
    ref = O.label_canonical(img, 0)
    compare_image(res.image(0), ref, "cfg3")
    depth = np.zeros(ref.n_components, dtype=np.int64)
    for c in range(1, ref.n_components):
        depth[c] = depth[ref.comps["parent"][c]] + 1
    assert depth.max() >= 8


def test_cfg4_sample(labeler):
    from paper_2006_09299_b200.runlab import cfg4_params
    idx = list(range(8)) + [97, 1023, 2048, 4095]
    imgs = np.stack([O.generate(1920, 1080, *cfg4_params(i), i) for i in idx])
    res = labeler.label_batch(imgs, LabelingConfig())
    for k, i in enumerate(idx):
        compare_image(res.image(k), O.label_canonical(imgs[k], 0), f"cfg4 #{i}")


@pytest.mark.timeout(900)
def test_cfg5_full(labeler):
    img = O.generate(32768, 32768, 0.45, 4, 5)
    res = labeler.label_batch(img[None], LabelingConfig())
    got = res.image(0)
    ref = O.label_canonical(img, 0)
    compare_image(got, ref, "cfg5")
    _invariants(got, img)


def test_uniform_and_extreme_cells_batch(labeler):
    """cfg2's extreme cells (d = 0, 0.05, 0.95, 1 at g = 1) as one batch of full-size images."""
    imgs = np.stack([O.generate(2048, 2048, d, 1, 1) for d in (0.0, 0.05, 0.95, 1.0)])
    res = labeler.label_batch(imgs, LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True))
    for i in range(imgs.shape[0]):
        compare_image(res.image(i), O.label_canonical(imgs[i], 0), f"extreme cell {i}")
