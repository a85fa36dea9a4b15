"""Stress of the lock-free union-find: the tile passes unite with atomicMin
and path halving whose interleaving depends on which CTAs run when.  The result must not:

* the same batch labeled repeatedly on one context gives identical bytes every time;
* contexts whose tile grid takes the tiles in permuted orders (RUNLAB_GPU_PERMUTE: CTA k gets
  tile k * m mod n) give the same bytes, and they equal the oracle.
"""
from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2006_09299_b200 import Labeler, LabelingConfig
from tests.parity_util import compare_image

pytestmark = pytest.mark.gpu

CELLS = [(0.3, 1), (0.45, 1), (0.5, 1), (0.6, 1), (0.75, 1), (0.45, 2), (0.55, 2), (0.45, 4), (0.6, 4),
         (0.5, 8), (0.05, 1), (0.95, 1)]
CFG = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True, relabel=True)


@pytest.fixture(scope="module")
def batch():
    return np.stack([O.generate(1024, 768, d, g, 17 + i) for i, (d, g) in enumerate(CELLS)])


def _digest(res) -> str:
    h = hashlib.sha256()
    for a in (res.n_components, res.n_fg, res.n_survivors, res.comp_offset, res.comps, res.top,
              res.filled_image, res.labels):
        if a is not None:
            h.update(np.ascontiguousarray(a).tobytes())
    surv = res.top == np.concatenate([np.arange(res.comp_offset[i + 1] - res.comp_offset[i], dtype=np.uint32)
                                      for i in range(len(res.n_components))])
    h.update(res.filled[surv].tobytes())
    return h.hexdigest()


def test_repeated_runs_identical(labeler, batch):
    first = _digest(labeler.label_batch(batch, CFG))
    for _ in range(7):
        assert _digest(labeler.label_batch(batch, CFG)) == first


@pytest.mark.parametrize("perm", [7, 101, 997])
def test_permuted_tile_order_identical(labeler, batch, perm):
    want = labeler.label_batch(batch, CFG)
    os.environ["RUNLAB_GPU_PERMUTE"] = str(perm)
    try:
        lab = Labeler(0)
    finally:
        del os.environ["RUNLAB_GPU_PERMUTE"]
    try:
        got = lab.label_batch(batch, CFG)
    finally:
        lab.close()
    assert _digest(got) == _digest(want)
    if perm == 7:
        for i in range(batch.shape[0]):
            compare_image(got.image(i), O.label_canonical(batch[i], 0), f"perm {perm} #{i}")


def test_split_pipelines_identical(labeler):
    """rl_label_device of a large batch as 1, 2, 3 and 4 concurrent interleaved pipelines
    (rl_set_pipelines): identical bytes, hole-filled image included (also as P4 rows)."""
    import torch
    from paper_2006_09299_b200 import _native as N
    from paper_2006_09299_b200.runlab import generate_device
    W, H, B = 1024, 768, 96  # 75 Mpx: above the split threshold
    imgs = torch.empty((B, H, W), dtype=torch.uint8, device="cuda")
    for i in range(B):
        d, g = CELLS[i % len(CELLS)]
        generate_device(imgs[i].data_ptr(), W, H, d, g, 100 + i)
    torch.cuda.synchronize()
    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    digests = []
    for k in (1, 2, 3, 4):
        labeler.set_pipelines(k)
        labeler.label_device(imgs.data_ptr(), W, H, B, cfg)
        res = labeler.fetch()
        digests.append(_digest(res))
    labeler.set_pipelines(3)
    assert len(set(digests)) == 1
    ref = O.label_canonical(imgs[5].cpu().numpy(), 0)
    compare_image(res.image(5), ref, "split #5")


def test_concurrent_contexts_on_host_threads():
    """One context per host thread (the reference allows distinct images to be
    labeled concurrently): four threads label different batches at the same time,
    through rl_label and through rl_label_into, each result bit-exact against the oracle."""
    import threading

    import torch
    from oracle import oracle as O
    from paper_2006_09299_b200 import Labeler, LabelingConfig
    from tests.parity_util import compare_image
    from tests.test_gpu_into import _cap, _check, _into

    cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
    errors: list[str] = []

    def work(k: int):
        try:
            lab = Labeler(0)
            try:
                for rep in range(3):
                    imgs = np.stack([O.generate(700 + 13 * k, 300 + 7 * rep, 0.2 + 0.15 * k, 1 + (i + k) % 4,
                                                1000 * k + 10 * rep + i) for i in range(6)])
                    res = lab.label_batch(imgs, cfg)
                    for i in range(imgs.shape[0]):
                        compare_image(res.image(i), O.label_canonical(imgs[i], 0), f"thread {k} rep {rep} #{i}")
                    h_in = torch.from_numpy(imgs).pin_memory()
                    o, outs = _into(lab, h_in, cfg, rep % 2, _cap(res))
                    _check(o, outs, res, rep % 2)
            finally:
                lab.close()
        except Exception as e:  # noqa: BLE001 -- reported on the main thread
            errors.append(f"thread {k}: {type(e).__name__}: {e}")

    threads = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
