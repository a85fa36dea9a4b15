"""Seeded random shapes, densities, granularities and connectivities in mixed batches: every
output of the device path against the oracle, bit for bit (ragged tiles in both directions,
1-pixel-wide and -tall images, P4 input for a third of the batches)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2006_09299_b200 import LabelingConfig, _native as N
from paper_2006_09299_b200.runlab import pack_p4
from tests.parity_util import compare_image

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_batches(labeler, seed):
    rng = np.random.default_rng(1000 + seed)
    w = int(rng.choice([1, 2, 7, 31, 32, 33, 255, 256, 257, 300, 511, 777]))
    h = int(rng.choice([1, 3, 31, 32, 33, 64, 65, 100, 200]))
    n = int(rng.integers(1, 6))
    conn = int(rng.integers(0, 2))
    imgs = np.stack([O.generate(w, h, float(rng.random()), int(rng.integers(1, min(w, h, 8) + 1)),
                                int(rng.integers(0, 1 << 30))) for _ in range(n)])
    cfg = LabelingConfig(connectivity=conn, compute_features=True, compute_euler=True, fill_holes=True,
                         relabel=True)
    if seed % 3 == 2:  # P4 input through the device path
        d = torch.from_numpy(pack_p4(imgs).reshape(-1).copy()).cuda()
        labeler.label_device(d.data_ptr(), w, h, n, cfg, pixel_format=N.RL_PIXELS_P4)
        labeler.sync()
        res = labeler.fetch()
    else:
        res = labeler.label_batch(imgs, cfg)
    for i in range(n):
        want = O.label_canonical(imgs[i], conn, want_labels=True)
        # with fill_holes the label image holds post-fill roots (labeling.hpp:224-250 after the
        # fill closure); the oracle's labels are pre-fill canonical ids
        want.labels = want.top[want.labels]
        compare_image(res.image(i), want, f"seed={seed} {w}x{h} conn={conn} image {i}")
