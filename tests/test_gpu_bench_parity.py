"""Parity on the configurations exactly as bench.py times them (VERDICT r01 "weak" #1).

* cfg2: all 105 images generated on the device and labeled by ONE `label_device` call (the
  bench's step), every image compared with the reference compiled from its own headers
  (oracle/_ref; the C restatement where it is absent).
* cfg4: all 4096 images, in device-generated chunks of 512 (8 label_device calls).
* cfg5: the unsplit 1-Gpixel image against the reference itself, and cut into 8 in-process
  strips at full size against the unsplit result.
* cfg5-shaped strips across two real processes: the rank phases of `label_strip` with the
  four collectives over gloo (host-staged), against the oracle.

The reference runs on a pool of host threads (its ctypes calls release the GIL).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2006_09299_b200 import Labeler, LabelingConfig
from paper_2006_09299_b200.runlab import cfg2_cells, cfg4_params, generate_device
from tests.parity_util import compare_image

pytestmark = pytest.mark.gpu

FULL = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True)
THREADS = max(1, min(32, len(os.sched_getaffinity(0))))


def _reference(img: np.ndarray):
    return O.ref_label_canonical(img, 0) if O.ref_available() else O.label_canonical(img, 0)


def _check_batch(res, specs, W, H, tag, offset=0):
    """Every image of a device batch against the reference on the host (thread pool)."""

    def one(k):
        d, g, seed = specs[k]
        compare_image(res.image(k), _reference(O.generate(W, H, d, g, seed)), f"{tag} #{offset + k}")

    with ThreadPoolExecutor(THREADS) as ex:
        list(ex.map(one, range(len(specs))))


def _device_batch(specs, W, H):
    imgs = torch.empty((len(specs), H, W), dtype=torch.uint8, device="cuda")
    for i, (d, g, seed) in enumerate(specs):
        generate_device(imgs[i].data_ptr(), W, H, d, g, seed)
    torch.cuda.synchronize()
    return imgs


@pytest.mark.timeout(900)
def test_cfg2_one_call_all_105(labeler):
    specs = [(d, g, 1) for d, g in cfg2_cells()]
    imgs = _device_batch(specs, 2048, 2048)
    labeler.label_device(imgs.data_ptr(), 2048, 2048, len(specs), FULL)
    res = labeler.fetch()
    assert res.n_components.shape[0] == 105
    _check_batch(res, specs, 2048, 2048, "cfg2")


@pytest.mark.timeout(1800)
def test_cfg4_all_4096(labeler):
    W, H, CH = 1920, 1080, 512
    for c0 in range(0, 4096, CH):
        specs = [cfg4_params(i) + (i,) for i in range(c0, c0 + CH)]
        imgs = _device_batch(specs, W, H)
        labeler.label_device(imgs.data_ptr(), W, H, CH, FULL)
        res = labeler.fetch()
        del imgs
        _check_batch(res, specs, W, H, "cfg4", c0)


@pytest.fixture(scope="module")
def cfg5():
    W = H = 32768
    dev = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    generate_device(dev.data_ptr(), W, H, 0.45, 4, 5)
    torch.cuda.synchronize()
    yield dev
    del dev


@pytest.mark.timeout(1200)
def test_cfg5_unsplit_vs_reference(labeler, cfg5):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    labeler.label_device(cfg5.data_ptr(), 32768, 32768, 1, FULL)
    got = labeler.fetch().image(0)
    compare_image(got, O.ref_label_canonical(cfg5.cpu().numpy(), 0), "cfg5 vs reference")


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("driver", ["lockstep", "native"])
def test_cfg5_eight_strips_full_size(labeler, cfg5, driver):
    """Config 5 in 8 full-size strips: the Python lockstep driver, and the library's own
    single-call driver (rl_label_strips: host thread per strip, device-to-device collectives)."""
    from paper_2006_09299_b200.strips import concat, label_strips_in_process, label_strips_native, strip_rows
    W = H = 32768
    labeler.label_device(cfg5.data_ptr(), W, H, 1, FULL)
    whole = labeler.fetch().image(0)
    rows = strip_rows(H, 8)
    labs = [Labeler(0) for _ in range(8)]
    ptrs = [cfg5.data_ptr() + y0 * W for y0, _ in rows]
    try:
        if driver == "native":
            got = concat(label_strips_native(labs, ptrs, W, H, FULL))
        else:
            got = concat(label_strips_in_process(labs, ptrs, W, H, rows, FULL))
    finally:
        for lab in labs:
            lab.close()
    for k in ("n_components", "n_fg", "n_holes", "euler", "n_survivors"):
        assert got[k] == whole[k], k
    assert got["comps"].tobytes() == whole["comps"].tobytes()
    np.testing.assert_array_equal(got["top"], whole["top"])
    surv = whole["top"] == np.arange(whole["n_components"], dtype=np.uint32)
    assert got["filled"][surv].tobytes() == whole["filled"][surv].tobytes()
    assert np.array_equal(got["filled_image"], whole["filled_image"])


# ---------------------------------------------------------------- two real strip processes
def _strip_rank(rank, world, port, W, H, d, g, seed, q):
    import torch.distributed as dist

    from paper_2006_09299_b200.runlab import generate_rows_device
    from paper_2006_09299_b200.strips import HostStagedCollectives, label_strip, strip_rows
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        y0, h = strip_rows(H, world)[rank]
        strip = torch.empty((h, W), dtype=torch.uint8, device="cuda")
        generate_rows_device(strip.data_ptr(), W, H, y0, h, d, g, seed)
        lab = Labeler(0)
        coll = HostStagedCollectives()
        cfg = LabelingConfig(compute_features=True, compute_euler=True, fill_holes=True, relabel=True)
        label_strip(lab, strip.data_ptr(), W, H, y0, h, cfg, coll, fetch=False)  # warm, then reuse
        r = label_strip(lab, strip.data_ptr(), W, H, y0, h, cfg, coll, fetch=True)
        out = dict(rank=rank, y0=r.y0, n_components=r.n_components, n_fg=r.n_fg, n_holes=r.n_holes,
                   euler=r.euler, n_survivors=r.n_survivors, comp_lo=r.comp_lo, comp_hi=r.comp_hi,
                   comps=r.comps.copy(), top=r.top.copy(), filled=r.filled.copy(),
                   filled_image=r.filled_image.copy(), labels=r.labels.copy())
        lab.close()
        dist.destroy_process_group()
        q.put(out)
    except Exception as exc:  # pragma: no cover - reported by the parent
        import traceback
        q.put(dict(rank=rank, error=f"{exc!r}\n{traceback.format_exc()}"))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,W,H,d,g,seed", [(2, 2048, 1536, 0.45, 4, 5), (3, 1000, 700, 0.55, 1, 9)])
def test_strips_across_processes(world, W, H, d, g, seed):
    """label_strip + the real collective sequence in `world` processes (gloo, host-staged; the
    processes share the one GPU, no kernel waits on another process) == the oracle."""
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_strip_rank, args=(r, world, port, W, H, d, g, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted((q.get(timeout=500) for _ in procs), key=lambda o: o["rank"])
    for p in procs:
        p.join(60)
    errs = [o["error"] for o in outs if "error" in o]
    assert not errs, errs[0]
    ref = O.label_canonical(O.generate(W, H, d, g, seed), 0, want_labels=True)
    # ranks own consecutive canonical-id ranges; concatenated they are the whole image
    assert outs[0]["comp_lo"] == 0 and outs[-1]["comp_hi"] == ref.n_components
    assert all(a["comp_hi"] == b["comp_lo"] for a, b in zip(outs, outs[1:]))
    got = dict(n_components=outs[0]["n_components"], n_fg=outs[0]["n_fg"], n_holes=outs[0]["n_holes"],
               euler=outs[0]["euler"], n_survivors=outs[0]["n_survivors"],
               comps=np.concatenate([o["comps"] for o in outs]), top=np.concatenate([o["top"] for o in outs]),
               filled=np.concatenate([o["filled"] for o in outs]),
               filled_image=np.concatenate([o["filled_image"] for o in outs], axis=0))
    compare_image(got, ref, f"{world} processes")
    # relabel with fill: every pixel carries its post-fill root (labeling.hpp:224-250)
    labels = np.concatenate([o["labels"] for o in outs], axis=0)
    assert np.array_equal(labels, ref.top[ref.labels])
