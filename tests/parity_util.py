"""Shared comparison helpers for the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np


def compare_image(got: dict, ref, where: str = "") -> None:
    """Bit-exact comparison of one image's GPU result (BatchResult.image()) with the oracle's
    canonical result (oracle.Canonical)."""
    tag = f"[{where}] " if where else ""
    assert got["n_components"] == ref.n_components, f"{tag}C_pre {got['n_components']} != {ref.n_components}"
    assert got["n_fg"] == ref.n_fg, f"{tag}n_fg {got['n_fg']} != {ref.n_fg}"
    assert got["n_holes"] == ref.n_holes, f"{tag}n_holes"
    assert got["euler"] == ref.euler, f"{tag}euler"
    assert got["n_survivors"] == ref.n_survivors, f"{tag}C_post {got['n_survivors']} != {ref.n_survivors}"
    gc, rc = got["comps"], ref.comps
    if not np.array_equal(gc, rc):
        bad = np.nonzero(gc != rc)[0]
        i = int(bad[0])
        raise AssertionError(f"{tag}{bad.size} component records differ; first id {i}: "
                             f"gpu {gc[i]} ref {rc[i]}")
    if not np.array_equal(got["top"], ref.top):
        bad = np.nonzero(got["top"] != ref.top)[0]
        raise AssertionError(f"{tag}{bad.size} post-fill roots differ; first id {int(bad[0])}: "
                             f"gpu {got['top'][bad[0]]} ref {ref.top[bad[0]]}")
    surv = ref.top == np.arange(ref.n_components, dtype=np.uint32)
    gf, rf = got["filled"][surv], ref.filled[surv]
    if not np.array_equal(gf, rf):
        bad = np.nonzero(gf != rf)[0]
        ids = np.nonzero(surv)[0][bad]
        raise AssertionError(f"{tag}{bad.size} post-fill features differ; first id {int(ids[0])}: "
                             f"gpu {gf[bad[0]]} ref {rf[bad[0]]}")
    if not np.array_equal(got["filled_image"], ref.filled_image):
        n = int((got["filled_image"] != ref.filled_image).sum())
        raise AssertionError(f"{tag}filled image differs at {n} pixels")
    if ref.labels is not None and got.get("labels") is not None:
        if not np.array_equal(got["labels"], ref.labels):
            n = int((got["labels"] != ref.labels).sum())
            raise AssertionError(f"{tag}label image differs at {n} pixels")
