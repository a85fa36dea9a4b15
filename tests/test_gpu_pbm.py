"""P4 rasters read and written by the tile kernels (RL_PIXELS_P4) against the byte-per-pixel
path, and `runlab fill` on PBM files against the reference's fill + write_pbm."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2006_09299_b200 import Labeler, LabelingConfig, _native as N
from paper_2006_09299_b200.runlab import pack_p4, unpack_p4

pytestmark = pytest.mark.gpu

CFG = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True, relabel=True)


def _device_run(labeler, buf_u8, w, h, n, fmt):
    from paper_2006_09299_b200.strips import _DevArray
    d = torch.from_numpy(np.ascontiguousarray(buf_u8).reshape(-1)).cuda()
    labeler.label_device(d.data_ptr(), w, h, n, CFG, pixel_format=fmt)
    labeler.sync()
    res = labeler.fetch()
    # the filled image in the call's pixel format, straight from the device buffer
    rowb = (w + 7) // 8 if fmt == N.RL_PIXELS_P4 else w
    src = N.load().rl_device_filled_image(labeler.ctx)
    view = torch.as_tensor(_DevArray(src, n * h * rowb, "|u1"), device="cuda")
    return res, view.cpu().numpy().reshape(n, h, rowb)


@pytest.mark.parametrize("w,h", [(2048, 512), (1000, 300), (37, 11), (1, 5), (257, 64), (31, 40), (1920, 108)])
def test_p4_matches_u8(labeler, w, h):
    imgs = np.stack([O.generate(w, h, d, min(g, w, h), 3 + i) for i, (d, g) in enumerate([(0.5, 1), (0.3, 2), (0.7, 4)])])
    n = imgs.shape[0]
    rows = pack_p4(imgs)
    if w % 8:  # pad bits set to 1 must be ignored (io.hpp:76-77)
        rows[..., -1] |= np.uint8((1 << (8 - w % 8)) - 1)
    a = labeler.label_batch(imgs, CFG)
    b, filled_rows = _device_run(labeler, rows, w, h, n, N.RL_PIXELS_P4)
    for f in ("n_components", "n_fg", "n_holes", "n_survivors", "comp_offset"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
    assert a.comps.tobytes() == b.comps.tobytes()
    np.testing.assert_array_equal(a.top, b.top)
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_array_equal(filled_rows, pack_p4(a.filled_image))  # zero pad bits
    np.testing.assert_array_equal(unpack_p4(filled_rows, w), a.filled_image)


def test_p4_label_into_chunked(labeler):
    w, h, n = 2048, 2048, 12  # 8 + 4 images per chunk
    imgs = np.stack([O.generate(w, h, 0.05 + 0.08 * i, 1 + i % 4, 50 + i) for i in range(n)])
    rows = torch.from_numpy(pack_p4(imgs)).pin_memory()
    a = labeler.label_batch(imgs, LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True))
    total = int(a.comp_offset[-1])
    fill = torch.zeros(rows.shape, dtype=torch.uint8).pin_memory()
    comps = torch.zeros(total * 48, dtype=torch.uint8).pin_memory()
    summ = torch.zeros(n * 5, dtype=torch.int64).pin_memory()
    outs = N.RlHostOutputs(fill.data_ptr(), None, comps.data_ptr(), None, None, total, summ.data_ptr(), None,
                           0, 0, 0, 0, 0)
    labeler.label_into(rows.data_ptr(), w, h, n, LabelingConfig(compute_features=True, compute_euler=True,
                                                               fill_holes=True), outs, pixel_format=N.RL_PIXELS_P4)
    assert outs.h2d_bytes == rows.numel()
    np.testing.assert_array_equal(fill.numpy(), pack_p4(a.filled_image))
    assert comps.numpy().tobytes() == a.comps.tobytes()
    np.testing.assert_array_equal(summ.numpy().reshape(n, 5)[:, 0], a.n_components)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("p1", [False, True])
def test_fill_pbm_matches_reference_cli(labeler, p1):
    """`runlab fill in.pbm out.pbm` (tools/runlab.cpp:128-137): read_pbm, label_image with
    fill, binarize_labels, write_pbm P4."""
    for (w, h, d, g) in [(333, 200, 0.55, 1), (64, 64, 0.45, 2), (1024, 768, 0.5, 4)]:
        img = O.generate(w, h, d, g, 9)
        data = O.ref_write_pbm(img, p1=p1)
        want = O.ref_write_pbm(O.label_canonical(img, 0).filled_image)
        assert labeler.fill_pbm(data) == want


def test_fill_pbm_rejects_truncated(labeler):
    from paper_2006_09299_b200.runlab import PbmParseError
    with pytest.raises(PbmParseError) as e:
        labeler.fill_pbm(b"P4\n9 2\n\x80\xff")
    assert e.value.byte_offset == 9  # bytes.size(): io.hpp:104-106
