"""§8(e): one image cut into horizontal strips, each strip on its own context, against the
single-image pipeline (which the other GPU tests pin to the oracle) -- bit-exact tables, filled
image and labels, for several strip counts, ragged last strips, both connectivities, nested
holes spanning cuts and a percolating noise image."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2006_09299_b200 import Labeler, LabelingConfig
from paper_2006_09299_b200.runlab import generate_device, generate_rings_device
from paper_2006_09299_b200.strips import concat, label_strips_in_process, strip_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def labelers():
    labs = [Labeler(0) for _ in range(8)]
    yield labs
    for lab in labs:
        lab.close()


def _compare(got: dict, ref, label: str):
    im = ref.image(0)
    assert got["n_components"] == im["n_components"], label
    assert got["n_fg"] == im["n_fg"], label
    assert got["n_holes"] == im["n_holes"], label
    assert got["euler"] == im["euler"], label
    assert got["n_survivors"] == im["n_survivors"], label
    assert got["comps"].shape[0] == im["n_components"], label
    bad = np.nonzero(got["comps"] != im["comps"])[0]
    assert bad.size == 0, f"{label}: comps differ at {bad[:10]}"
    np.testing.assert_array_equal(got["top"], im["top"], err_msg=label)
    surv = im["top"] == np.arange(im["n_components"], dtype=np.uint32)
    assert got["filled"][surv].tobytes() == im["filled"][surv].tobytes(), label
    np.testing.assert_array_equal(got["filled_image"], im["filled_image"], err_msg=label)
    if "labels" in got:
        np.testing.assert_array_equal(got["labels"], im["labels"], err_msg=label)


def _run(labelers, img_dev, W, H, n, cfg):
    rows = strip_rows(H, n)
    ptrs = [img_dev.data_ptr() + y0 * W for (y0, _) in rows]
    return concat(label_strips_in_process(labelers[:n], ptrs, W, H, rows, cfg))


CASES = [(0.5, 1), (0.45, 4), (0.3, 2), (0.7, 1), (0.6, 8), (0.05, 1), (0.95, 1)]


@pytest.mark.parametrize("d,g", CASES)
@pytest.mark.parametrize("n", [2, 3, 5])
def test_strips_match_single_image(labelers, labeler, d, g, n):
    W, H = 1536, 1000  # ragged last strip, 6 tile columns
    img = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    generate_device(img.data_ptr(), W, H, d, g, 7)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    ref = labeler.label_batch(img.cpu().numpy()[None], cfg)
    _compare(_run(labelers, img, W, H, n, cfg), ref, f"d={d} g={g} n={n}")


@pytest.mark.parametrize("conn", [0, 1])
def test_strips_rings_and_labels(labelers, labeler, conn):
    W = H = 1024
    img = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    generate_rings_device(img.data_ptr(), W, H, 64, 3, 0.02)
    cfg = LabelingConfig(connectivity=conn, compute_features=True, compute_euler=True, fill_holes=True,
                         relabel=True)
    ref = labeler.label_batch(img.cpu().numpy()[None], cfg)
    _compare(_run(labelers, img, W, H, 4, cfg), ref, f"rings conn={conn}")


def test_strips_nested_shapes_across_cuts(labelers, labeler):
    """Concentric square rings centred on a cut: every ring, hole and the fill cross strips."""
    W, H = 512, 256
    img = np.zeros((H, W), dtype=np.uint8)
    for k in range(0, 60, 3):
        img[128 - 100 + k:128 + 100 - k, 256 - 200 + 2 * k:256 + 200 - 2 * k] = (k // 3) % 2 == 0
    img[0, :] = 1  # a component touching the top frame only
    img[:, 0] = 0
    dev = torch.from_numpy(img).cuda()
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True, relabel=True)
    ref = labeler.label_batch(img[None], cfg)
    for n in (2, 4, 8):
        _compare(_run(labelers, dev, W, H, n, cfg), ref, f"nested n={n}")


def test_strips_uniform_images(labelers, labeler):
    W, H = 300, 200
    for v in (0, 1):
        img = np.full((H, W), v, dtype=np.uint8)
        dev = torch.from_numpy(img).cuda()
        cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True, relabel=True)
        ref = labeler.label_batch(img[None], cfg)
        _compare(_run(labelers, dev, W, H, 3, cfg), ref, f"uniform {v}")


def test_strips_against_oracle(labelers):
    W, H = 777, 300
    img = O.generate(W, H, 0.55, 1, 3)
    dev = torch.from_numpy(img).cuda()
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    got = _run(labelers, dev, W, H, 4, cfg)
    want = O.label_canonical(img, 0)
    assert got["n_components"] == want.n_components
    assert got["comps"].tobytes() == want.comps.tobytes()
    np.testing.assert_array_equal(got["filled_image"], want.filled_image)


def test_strips_reject_densify(labelers):
    img = torch.zeros((64, 64), dtype=torch.uint8, device="cuda")
    cfg = LabelingConfig(relabel=True, densify_labels=True, fill_holes=True)
    with pytest.raises(ValueError):
        _run(labelers, img, 64, 64, 2, cfg)


def test_generate_rows_matches_full():
    from paper_2006_09299_b200.runlab import generate_rows_device
    W, H = 1000, 700
    full = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    generate_device(full.data_ptr(), W, H, 0.45, 4, 5)
    for y0, h in strip_rows(H, 3):
        part = torch.empty((h, W), dtype=torch.uint8, device="cuda")
        generate_rows_device(part.data_ptr(), W, H, y0, h, 0.45, 4, 5)
        assert torch.equal(part, full[y0:y0 + h])


def test_strips_poisoned_workspace(labeler):
    """Fresh contexts whose workspaces start filled with a pattern instead of zeros (recycled
    device memory): every table the strip phases read must have been written first."""
    import os
    os.environ["RUNLAB_GPU_POISON"] = "1"
    labs = [Labeler(0) for _ in range(3)]
    try:
        W, H = 1536, 1000
        img = torch.empty((H, W), dtype=torch.uint8, device="cuda")
        cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True, relabel=True)
        for d, g in ((0.5, 1), (0.45, 4)):
            generate_device(img.data_ptr(), W, H, d, g, 11)
            ref = labeler.label_batch(img.cpu().numpy()[None], cfg)
            _compare(_run(labs, img, W, H, 3, cfg), ref, f"poisoned d={d} g={g}")
    finally:
        del os.environ["RUNLAB_GPU_POISON"]
        for lab in labs:
            lab.close()


def test_strip_workspace_follows_the_strip(labeler):
    """A strip context's device tables are sized by its strip: tile tables, cells,
    nodes and component tables hold the strip's share, not the whole image's."""
    W = H = 8192
    img = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    generate_device(img.data_ptr(), W, H, 0.45, 4, 5)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    whole = Labeler(0)
    labs = [Labeler(0) for _ in range(8)]
    try:
        whole.label_device(img.data_ptr(), W, H, 1, cfg)
        ref = whole.fetch()
        full = whole.workspace_bytes()
        got = _run(labs, img, W, H, 8, cfg)
        _compare(got, ref, "8192^2 in 8 strips")
        per = [lab.workspace_bytes() for lab in labs]
        assert max(per) < 0.3 * full, (per, full)
    finally:
        whole.close()
        for lab in labs:
            lab.close()


# ---- the library's single-call driver (rl_label_strips): strips on several contexts of one
# process, collectives as device-to-device copies + reduction kernels
def _run_native(labelers, img_dev, W, H, n, cfg):
    from paper_2006_09299_b200.strips import label_strips_native
    rows = strip_rows(H, n)
    ptrs = [img_dev.data_ptr() + y0 * W for (y0, _) in rows]
    return concat(label_strips_native(labelers[:n], ptrs, W, H, cfg))


@pytest.mark.parametrize("d,g", [(0.5, 1), (0.45, 4), (0.95, 1)])
@pytest.mark.parametrize("n", [1, 2, 5, 8])
def test_native_strips_match_single_image(labelers, labeler, d, g, n):
    W, H = 1536, 1000
    img = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    generate_device(img.data_ptr(), W, H, d, g, 11)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    labeler.label_device(img.data_ptr(), W, H, 1, cfg)
    labeler.sync()
    ref = labeler.fetch()
    _compare(_run_native(labelers, img, W, H, n, cfg), ref, f"native d={d} g={g} n={n}")
    # repeated calls reuse the contexts' exchange buffers
    _compare(_run_native(labelers, img, W, H, n, cfg), ref, f"native again d={d} g={g} n={n}")


def test_native_strips_rings_labels_and_oracle(labelers):
    W, H = 777, 300
    img = O.generate_rings(W, H, 64, 3, 0.02)
    dev = torch.from_numpy(img).cuda()
    for conn in (0, 1):
        ref = O.label_canonical(img, conn, want_labels=True)
        cfg = LabelingConfig(connectivity=conn, compute_features=True, compute_euler=True, fill_holes=True)
        got = _run_native(labelers, dev, W, H, 4, cfg)
        assert got["n_components"] == ref.n_components and got["euler"] == ref.euler
        assert got["comps"].tobytes() == ref.comps.tobytes()
        np.testing.assert_array_equal(got["top"], ref.top)
        np.testing.assert_array_equal(got["filled_image"], ref.filled_image)
        # the label image (pre-fill canonical ids, Alg. 4 relabel)
        cfg = LabelingConfig(connectivity=conn, compute_features=True, relabel=True)
        got = _run_native(labelers, dev, W, H, 4, cfg)
        np.testing.assert_array_equal(got["labels"], ref.labels)


def test_native_strip_rows_and_errors(labelers):
    import ctypes as C
    from paper_2006_09299_b200.strips import label_strips_native
    L = labelers[0]._L
    y0, h = (C.c_int32 * 5)(), (C.c_int32 * 5)()
    assert L.rl_strip_rows(1000, 5, y0, h) == 0
    assert [(a, b) for a, b in zip(y0, h)] == strip_rows(1000, 5)
    assert L.rl_strip_rows(64, 3, y0, h) != 0  # more strips than tile rows
    img = torch.zeros((64, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(Exception):
        label_strips_native(labelers[:3], [img.data_ptr()] * 3, 64, 64, LabelingConfig())


@pytest.mark.parametrize("seed", range(1, 9))
def test_strips_structured_fuzz(labelers, seed):
    """Bands of adversarial row patterns (tools/fuzz_struct.py) cut into 2-6 strips at rows that
    fall inside the bands (events, merge rows and checkerboards across the cuts), against the
    oracle: every table, the filled image and the label image."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_struct as F
    rng = np.random.default_rng(100 + seed)
    W, H = int(rng.choice([2048, 1537, 700])), int(rng.choice([600, 333, 1000]))
    img = F.image(rng, W, H)
    conn = int(rng.integers(0, 2))
    n = int(rng.integers(2, 7))
    dev = torch.from_numpy(img).cuda()
    cfg = LabelingConfig(connectivity=conn, compute_features=True, compute_euler=True, fill_holes=True,
                         relabel=True)
    got = _run(labelers, dev, W, H, n, cfg)
    want = O.label_canonical(img, conn, want_labels=True)
    label = f"seed {seed} {W}x{H} conn {conn} strips {n}"
    assert got["n_components"] == want.n_components, label
    assert got["n_fg"] == want.n_fg and got["n_holes"] == want.n_holes and got["euler"] == want.euler, label
    assert got["n_survivors"] == want.n_survivors, label
    bad = np.nonzero(got["comps"] != want.comps)[0]
    assert bad.size == 0, f"{label}: comps differ at {bad[:10]}"
    np.testing.assert_array_equal(got["top"], want.top, err_msg=label)
    surv = want.top == np.arange(want.n_components, dtype=np.uint32)
    assert got["filled"][surv].tobytes() == want.filled[surv].tobytes(), label
    np.testing.assert_array_equal(got["filled_image"], want.filled_image, err_msg=label)
    # with hole filling the label image holds post-fill roots (labeling.hpp:231-236)
    np.testing.assert_array_equal(got["labels"], want.top[want.labels], err_msg=label)
