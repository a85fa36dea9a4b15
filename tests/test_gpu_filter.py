"""filter_components (analysis.hpp:89-125) on the device vs the oracle restatement (which
tests/test_oracle_pin.py pins to the reference's own filter_components)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2006_09299_b200 import LabelingConfig
from paper_2006_09299_b200.runlab import filter_components

pytestmark = pytest.mark.gpu


def _check(comps, sel, label):
    got = filter_components(comps, sel)
    want = O.filter_components(comps, sel)
    for k, (a, b) in enumerate(zip(got, want)):
        assert a.tobytes() == b.tobytes(), f"{label}: output {k} differs"


@pytest.mark.parametrize("d,g", [(0.5, 1), (0.3, 2), (0.45, 4), (0.7, 1), (0.6, 8)])
def test_filter_matches_oracle(labeler, d, g):
    img = O.generate(512, 384, d, g, 21)
    res = labeler.label_batch(img[None], LabelingConfig(compute_features=True, fill_holes=True))
    comps = res.image(0)["comps"]
    n = comps.shape[0]
    rng = np.random.default_rng(5)
    fg = (comps["flags"] & 1).astype(bool)
    sels = {"holes": (~fg) & (np.arange(n) > 0), "small fg": fg & (comps["s"] <= 4),
            "random": (rng.random(n) < 0.25) & (np.arange(n) > 0), "none": np.zeros(n, bool),
            "all": np.arange(n) > 0, "wide bbox": (comps["col_max"] - comps["col_min"] > 10) & (np.arange(n) > 0)}
    for name, sel in sels.items():
        _check(comps, sel, f"d={d} g={g} {name}")


def test_filter_holes_equals_fill(labeler):
    """test_analysis.cpp:146-210: filtering the holes is hole filling (device result vs device fill)."""
    img = O.generate_rings(1024, 1024, 64, 3, 0.02)
    res = labeler.label_batch(img[None], LabelingConfig(compute_features=True, fill_holes=True))
    im = res.image(0)
    n = im["n_components"]
    sel = ((im["comps"]["flags"] & 1) == 0) & (np.arange(n) > 0)
    parent, feats, _ = filter_components(im["comps"], sel)
    np.testing.assert_array_equal(parent, im["top"])
    surv = im["top"] == np.arange(n)
    assert feats[surv].tobytes() == im["filled"][surv].tobytes()


def test_filter_device_selection(labeler):
    """Predicate evaluated on the device (torch) over device-resident records."""
    img = O.generate(700, 500, 0.55, 2, 4)
    res = labeler.label_batch(img[None], LabelingConfig(compute_features=True))
    comps = res.image(0)["comps"]
    d = torch.from_numpy(comps.view(np.uint8).reshape(-1).copy()).cuda()
    s = d.view(torch.int64).view(-1, 6)[:, 0]  # S of each 48-B record
    sel = (s < 6)
    sel[0] = False
    got = filter_components(d, sel)
    want = O.filter_components(comps, sel.cpu().numpy())
    for a, b in zip(got, want):
        assert a.tobytes() == b.tobytes()


def test_filter_rejects_exterior(labeler):
    img = O.generate(64, 64, 0.5, 1, 1)
    comps = labeler.label_batch(img[None], LabelingConfig()).image(0)["comps"]
    sel = np.zeros(comps.shape[0], dtype=np.uint8)
    sel[0] = 1
    with pytest.raises(ValueError):
        filter_components(comps, sel)
