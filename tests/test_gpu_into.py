"""rl_label_into (the host-buffer entry point) against one whole-batch rl_label call.

Batches above ~32 Mpixel are cut into chunks of whole images that are pipelined through
several workspaces; every output must equal the single-pipeline result bit for bit (which the
other GPU tests pin to the oracle), for both layouts of the post-fill features.
"""
from __future__ import annotations

import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2006_09299_b200 import Labeler, LabelingConfig, _native as N
from paper_2006_09299_b200.runlab import generate_device

pytestmark = pytest.mark.gpu


def _batch(n, h, w, seed0=1):
    d = torch.empty((n, h, w), dtype=torch.uint8, device="cuda")
    for i in range(n):
        dens = 0.05 + 0.9 * ((i * 7) % 19) / 18.0
        generate_device(d[i].data_ptr(), w, h, dens, 1 + (i % 5), seed0 + i)
    torch.cuda.synchronize()
    return d.cpu().pin_memory()


@pytest.fixture(scope="module")
def small_chunks():
    """A context whose rl_label_into cuts batches into 1-Mpixel chunks."""
    os.environ["RUNLAB_GPU_CHUNK_PX"] = str(1 << 20)
    try:
        lab = Labeler(0)
    finally:
        del os.environ["RUNLAB_GPU_CHUNK_PX"]
    yield lab
    lab.close()


def _into(labeler, h_in, cfg, layout, cap, labels=False, expect_error=None):
    n, h, w = h_in.shape
    o = {
        "fill": torch.zeros((n, h, w), dtype=torch.uint8).pin_memory(),
        "summ": torch.zeros(n * 5, dtype=torch.int64).pin_memory(),
        "off": torch.zeros(n + 1, dtype=torch.int64).pin_memory(),
    }
    o["comps"] = torch.zeros(cap * 48, dtype=torch.uint8).pin_memory()
    o["top"] = torch.zeros(cap, dtype=torch.int32).pin_memory()
    o["filled"] = torch.zeros(cap * 40, dtype=torch.uint8).pin_memory()
    if labels:
        o["labels"] = torch.zeros((n, h, w), dtype=torch.int32).pin_memory()
    outs = N.RlHostOutputs(o["fill"].data_ptr(), o["labels"].data_ptr() if labels else None,
                           o["comps"].data_ptr(), o["top"].data_ptr(), o["filled"].data_ptr(), cap,
                           o["summ"].data_ptr(), o["off"].data_ptr(), 0, 0, 0, layout, 0)
    if expect_error is None:
        labeler.label_into(h_in.data_ptr(), w, h, n, cfg, outs)
    else:
        with pytest.raises(expect_error):
            labeler.label_into(h_in.data_ptr(), w, h, n, cfg, outs)
    return o, outs


def _check(o, outs, ref, layout, labels=False):
    n = ref.n_images
    total = int(ref.comp_offset[-1])
    assert outs.comps_needed == total
    summ = o["summ"].numpy().reshape(n, 5)
    np.testing.assert_array_equal(summ[:, 0], ref.n_components)
    np.testing.assert_array_equal(summ[:, 1], ref.n_fg)
    np.testing.assert_array_equal(summ[:, 2], ref.n_holes)
    np.testing.assert_array_equal(summ[:, 3], ref.euler)
    np.testing.assert_array_equal(summ[:, 4], ref.n_survivors)
    np.testing.assert_array_equal(o["off"].numpy(), ref.comp_offset)
    np.testing.assert_array_equal(o["fill"].numpy(), ref.filled_image)
    comps = o["comps"].numpy()[: total * 48].view(O.COMPONENT_DTYPE)
    assert comps.tobytes() == ref.comps.tobytes()
    top = o["top"].numpy()[:total].astype(np.uint32)
    np.testing.assert_array_equal(top, ref.top)
    # survivors: top[e] == e (image-relative ids)
    rel = np.concatenate([np.arange(ref.comp_offset[i + 1] - ref.comp_offset[i], dtype=np.uint32)
                          for i in range(n)])
    surv = top == rel
    assert int(surv.sum()) == int(ref.n_survivors.sum())
    if layout == 0:
        filled = o["filled"].numpy()[: total * 40].view(O.FEATURE_DTYPE)
        assert filled[surv].tobytes() == ref.filled[surv].tobytes()
    else:
        ns = int(surv.sum())
        filled = o["filled"].numpy()[: ns * 40].view(O.FEATURE_DTYPE)
        assert filled.tobytes() == ref.filled[surv].tobytes()
    if labels:
        np.testing.assert_array_equal(o["labels"].numpy().view(np.uint32), ref.labels)
    n_, h_, w_ = o["fill"].shape
    # byte-per-pixel input crosses as P4 bits unless RUNLAB_GPU_PACKED_H2D=0
    assert outs.h2d_bytes in (o["fill"].numel(), n_ * h_ * ((w_ + 7) // 8))


def _cap(ref):
    return int(ref.comp_offset[-1]) + 1024


@pytest.mark.parametrize("n", [3, 20, 41])
@pytest.mark.parametrize("layout", [0, 1])
def test_into_small_chunks(small_chunks, n, layout):
    h_in = _batch(n, 512, 512)  # 4 images per chunk
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    ref = small_chunks.label_batch(h_in.numpy(), cfg)
    for _ in range(2):  # the second call replays the chunk pipelines' graphs
        o, outs = _into(small_chunks, h_in, cfg, layout, _cap(ref))
        _check(o, outs, ref, layout)


@pytest.mark.parametrize("layout", [0, 1])
def test_into_default_chunks(labeler, layout):
    h_in = _batch(21, 2048, 2048)  # 8 + 8 + 5 images
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    ref = labeler.label_batch(h_in.numpy(), cfg)
    o, outs = _into(labeler, h_in, cfg, layout, _cap(ref))
    _check(o, outs, ref, layout)


def test_into_chunked_labels(small_chunks):
    h_in = _batch(10, 512, 512, seed0=77)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True, relabel=True)
    ref = small_chunks.label_batch(h_in.numpy(), cfg)
    o, outs = _into(small_chunks, h_in, cfg, 1, _cap(ref), labels=True)
    _check(o, outs, ref, 1, labels=True)


def test_into_enospc_reports_total(small_chunks):
    h_in = _batch(10, 512, 512, seed0=5)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    ref = small_chunks.label_batch(h_in.numpy(), cfg)
    o, outs = _into(small_chunks, h_in, cfg, 1, 1000, expect_error=RuntimeError)
    assert outs.comps_needed == int(ref.comp_offset[-1])
    np.testing.assert_array_equal(o["fill"].numpy(), ref.filled_image)  # still complete
    o, outs = _into(small_chunks, h_in, cfg, 1, _cap(ref))
    _check(o, outs, ref, 1)


def test_into_bad_layout(labeler):
    h_in = _batch(1, 64, 64)
    _into(labeler, h_in, LabelingConfig(), 2, 16, expect_error=ValueError)


def test_into_chunked_densified_labels(small_chunks):
    """densify_labels through the chunked path: ranks of post-fill roots per image."""
    h_in = _batch(9, 512, 512, seed0=31)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True, relabel=True,
                         densify_labels=True)
    ref = small_chunks.label_batch(h_in.numpy(), cfg)
    o, outs = _into(small_chunks, h_in, cfg, 0, _cap(ref), labels=True)
    _check(o, outs, ref, 0, labels=True)


@pytest.mark.parametrize("layout", [0, 1])
def test_into_packed_slots_match_full_records(small_chunks, layout):
    """Compact record/feature slots (pack.cuh) decode to exactly the full records.

    Dense noise gives many one-tile components (slots); solid and coarse images give
    components that span tiles, exteriors with s = 0 and features past the slot ranges
    (escapes).  A context with RUNLAB_GPU_NO_PACKED_RECORDS copies the full tables."""
    h_in = _batch(12, 512, 512, seed0=11)
    h_in[3].fill_(1)
    h_in[4].fill_(0)
    h_in[5, 100:400, 50:500] = 1
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    ref = small_chunks.label_batch(h_in.numpy(), cfg)
    o, outs = _into(small_chunks, h_in, cfg, layout, _cap(ref))
    _check(o, outs, ref, layout)
    os.environ["RUNLAB_GPU_NO_PACKED_RECORDS"] = "1"
    os.environ["RUNLAB_GPU_CHUNK_PX"] = str(1 << 20)
    try:
        plain = Labeler(0)
    finally:
        del os.environ["RUNLAB_GPU_NO_PACKED_RECORDS"]
        del os.environ["RUNLAB_GPU_CHUNK_PX"]
    try:
        o2, outs2 = _into(plain, h_in, cfg, layout, _cap(ref))
        _check(o2, outs2, ref, layout)
    finally:
        plain.close()
    total = int(ref.comp_offset[-1])
    assert outs.d2h_bytes < outs2.d2h_bytes - 20 * total  # 48-B records became 20-B slots


@pytest.mark.parametrize("env", [{"RUNLAB_GPU_PACKED_H2D": "0"}, {"RUNLAB_GPU_NO_PACKED_D2H": "1"},
                                 {"RUNLAB_GPU_NO_PACKED_D2H": "1", "RUNLAB_GPU_NO_PACKED_RECORDS": "1"}])
def test_into_copy_variants(env):
    """The chunked path with the u8 input copied plainly (no host-side P4 packing), and with the
    input packed but the filled image (and records) copied plainly: same outputs; the reported
    H2D bytes follow the input format on the link."""
    h_in = _batch(13, 512, 384, seed0=23)
    h_in[2].fill_(1)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    os.environ.update(env)
    os.environ["RUNLAB_GPU_CHUNK_PX"] = str(1 << 20)
    try:
        lab = Labeler(0)
    finally:
        for k in list(env) + ["RUNLAB_GPU_CHUNK_PX"]:
            del os.environ[k]
    try:
        ref = lab.label_batch(h_in.numpy(), cfg)
        for _ in range(2):
            o, outs = _into(lab, h_in, cfg, 1, _cap(ref))
            _check(o, outs, ref, 1)
        n, h, w = h_in.shape
        want = n * h * w if env.get("RUNLAB_GPU_PACKED_H2D") == "0" else n * h * ((w + 7) // 8)
        assert outs.h2d_bytes == want
    finally:
        lab.close()


# one chunk of at least RUNLAB_GPU_BIG_PX pixels (8 Mi by default) crosses PCIe packed: the
# input packed to P4 in row pieces copied as they are packed, the filled image expanded while
# the component tables cross
@pytest.mark.parametrize("shape", [(1, 2048, 4096), (2, 1500, 3000)])
@pytest.mark.parametrize("layout", [0, 1])
def test_into_one_large_chunk(labeler, shape, layout):
    n, h, w = shape
    h_in = _batch(n, h, w, seed0=31)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    ref = labeler.label_batch(h_in.numpy(), cfg)
    for _ in range(2):
        o, outs = _into(labeler, h_in, cfg, layout, _cap(ref))
        _check(o, outs, ref, layout)
        assert outs.h2d_bytes == n * h * ((w + 7) // 8)  # packed input


def test_into_one_large_chunk_labels(labeler):
    h_in = _batch(1, 2048, 4096, seed0=41)
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True, relabel=True)
    ref = labeler.label_batch(h_in.numpy(), cfg)
    o, outs = _into(labeler, h_in, cfg, 1, _cap(ref), labels=True)
    _check(o, outs, ref, 1, labels=True)
