"""GPU: the reference-generated golden fixtures, the Python mirror's reference-style API and the
C++ drop-in (include/runlab_gpu.hpp) running the reference's known-answer tests."""
from __future__ import annotations

import glob
import os
import subprocess

import numpy as np
import pytest

from tests.parity_util import compare_image

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "*.npz")))


class _Ref:
    def __init__(self, z):
        for k in z.files:
            setattr(self, k, z[k])
        for k in ("n_components", "n_fg", "n_holes", "euler", "n_survivors", "conn"):
            setattr(self, k, int(getattr(self, k)))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_gpu_matches_reference_goldens(labeler, path):
    from paper_2006_09299_b200 import Connectivity, LabelingConfig
    ref = _Ref(np.load(path))
    cfg = LabelingConfig(connectivity=Connectivity(ref.conn), relabel=True)
    res = labeler.label_batch(ref.image[None], cfg)
    compare_image(res.image(0), ref, os.path.basename(path))


def test_python_mirror_fig3(labeler):
    """test_labeling.cpp:107-148 through the Python mirror of label_image."""
    from paper_2006_09299_b200 import (LabelingConfig, adjacency_tree, binarize_labels, euler_number,
                                       holes, label_image)
    img = np.load(os.path.join(ROOT, "tests", "golden", "fig_example.npz"))["image"]
    cfg = LabelingConfig(compute_features=True, compute_euler=True, relabel=True)
    res = label_image(img, cfg, labeler)
    assert (res.fg_count, res.hole_count, res.euler) == (1, 1, 0)
    assert res.roots() == [0, 1, 2]
    assert int(res.adjacency[2]) == 1 and int(res.adjacency[1]) == 0
    assert int(res.features[1]["s"]) == 56 and int(res.features[2]["s"]) == 11
    assert list(res.labels[3]) == [0, 1, 0, 1, 2, 1, 0, 0, 0, 1, 2, 1, 0, 1, 0]
    assert [h.root for h in holes(res)] == [2] and euler_number(res) == 0
    assert adjacency_tree(res).children[0] == [1]
    cfg.fill_holes = True
    filled = label_image(img, cfg, labeler)
    assert filled.roots() == [0, 1] and int(filled.features[1]["s"]) == 67
    assert list(binarize_labels(filled.labels, filled.equivalences)[3]) == [0, 1, 0, 1, 1, 1, 0, 0, 0, 1, 1, 1, 0, 1, 0]


def test_densified_fill_labels_match_pixel_fill(labeler):
    """test_labeling.cpp:301-319: fill + relabel + densify == flood_label(oracle_fill_holes)."""
    from oracle import oracle as O
    from paper_2006_09299_b200 import Connectivity, LabelingConfig, label_image
    for conn in (0, 1):
        for seed in (51, 52, 53):
            img = O.generate(25, 25, 0.55, 1, seed)
            cfg = LabelingConfig(connectivity=Connectivity(conn), relabel=True, densify_labels=True,
                                 fill_holes=True)
            res = label_image(img, cfg, labeler)
            _, comp, _ = O.flood_label(O.fill_holes(img, conn), conn)
            assert np.array_equal(res.labels.astype(np.int32), comp)
    # larger, multi-tile
    img = O.generate(700, 300, 0.55, 1, 9)
    res = label_image(img, LabelingConfig(relabel=True, densify_labels=True, fill_holes=True), labeler)
    _, comp, _ = O.flood_label(O.fill_holes(img, 0), 0)
    assert np.array_equal(res.labels.astype(np.int32), comp)


def test_cpp_dropin_binary():
    import __graft_entry__ as ge
    binary = ge.build_cpp_dropin_test()
    out = subprocess.run([binary], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "PASS" in out.stdout
