"""ctypes front-end to the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs import this module.  It loads

* ``oracle/liboracle.so`` -- the plain-C restatement of the reference path
  (``oracle/runlab_oracle.c``), and
* ``oracle/_ref/libref_runlab.so`` -- the reference itself compiled from its unmodified
  headers (``oracle/ref_shim.cpp``; built only where ``/root/reference`` exists and shipped
  prebuilt to the GPU box).

Both return the canonical result layout shared with the GPU C ABI
(``include/runlab_gpu.h``): components numbered by raster order of their first pixel,
exterior = 0.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

FEATURE_DTYPE = np.dtype([("s", "<i8"), ("sx", "<i8"), ("sy", "<i8"), ("row_min", "<i4"),
                          ("row_max", "<i4"), ("col_min", "<i4"), ("col_max", "<i4")])
COMPONENT_DTYPE = np.dtype([("s", "<i8"), ("sx", "<i8"), ("sy", "<i8"), ("row_min", "<i4"),
                            ("row_max", "<i4"), ("col_min", "<i4"), ("col_max", "<i4"),
                            ("parent", "<u4"), ("flags", "<u4")])
assert FEATURE_DTYPE.itemsize == 40 and COMPONENT_DTYPE.itemsize == 48


class _OrcResult(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("n_components", C.c_int64),
                ("n_fg", C.c_int64), ("n_holes", C.c_int64), ("euler", C.c_int64),
                ("n_survivors", C.c_int64), ("comps", C.c_void_p), ("top", C.c_void_p),
                ("filled", C.c_void_p), ("filled_image", C.c_void_p), ("labels", C.c_void_p)]


@dataclass
class Canonical:
    """One image's canonical labeling (same fields as the GPU result)."""
    width: int
    height: int
    n_components: int
    n_fg: int
    n_holes: int
    euler: int
    n_survivors: int
    comps: np.ndarray         # COMPONENT_DTYPE [n_components]
    top: np.ndarray           # uint32 [n_components]
    filled: np.ndarray        # FEATURE_DTYPE [n_components]; valid where top == arange
    filled_image: np.ndarray  # uint8 [h, w]
    labels: np.ndarray | None # uint32 [h, w]


def _copy(ptr, dtype, n):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    buf = (C.c_char * (n * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(bytes(buf), dtype=dtype).copy()


def _to_canonical(r: _OrcResult, want_labels: bool) -> Canonical:
    n = r.n_components
    w, h = r.width, r.height
    return Canonical(
        width=w, height=h, n_components=n, n_fg=r.n_fg, n_holes=r.n_holes, euler=r.euler,
        n_survivors=r.n_survivors,
        comps=_copy(r.comps, COMPONENT_DTYPE, n),
        top=_copy(r.top, np.uint32, n),
        filled=_copy(r.filled, FEATURE_DTYPE, n),
        filled_image=_copy(r.filled_image, np.uint8, w * h).reshape(h, w),
        labels=_copy(r.labels, np.uint32, w * h).reshape(h, w) if want_labels else None)


_lib = None
_ref = None


def lib():
    """The C restatement (oracle/liboracle.so)."""
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or build())")
        L = C.CDLL(path)
        L.orc_block_draw.restype = C.c_uint64
        L.orc_block_draw.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_generate.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_uint64, C.c_void_p]
        L.orc_generate_rings.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_void_p]
        L.orc_cfg4_params.argtypes = [C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        L.orc_encode_row.restype = C.c_int32
        L.orc_encode_row.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        L.orc_label_canonical.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int, C.c_int,
                                          C.POINTER(_OrcResult)]
        L.orc_result_free.argtypes = [C.POINTER(_OrcResult)]
        L.orc_flood_label.restype = C.c_int32
        L.orc_flood_label.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_int32]
        L.orc_bitquad_euler.restype = C.c_int64
        L.orc_bitquad_euler.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int]
        L.orc_fill_holes.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int, C.c_void_p]
        L.orc_filter_components.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_void_p]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libref_runlab.so"))


def ref():
    """The reference compiled from its own headers (oracle/_ref/libref_runlab.so)."""
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libref_runlab.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build it with `make -C oracle ref` "
                                    "where /root/reference exists")
        L = C.CDLL(path)
        L.ref_generate.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_uint64, C.c_void_p]
        L.ref_encode_row.restype = C.c_int32
        L.ref_encode_row.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        L.ref_label_canonical.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int, C.c_int,
                                          C.POINTER(_OrcResult)]
        L.ref_result_free.argtypes = [C.POINTER(_OrcResult)]
        L.ref_flood_label.restype = C.c_int32
        L.ref_flood_label.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int, C.c_void_p]
        L.ref_bitquad_euler.restype = C.c_int64
        L.ref_bitquad_euler.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int]
        L.ref_filter_components.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int, C.c_void_p,
                                             C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_read_pbm.argtypes = [C.c_char_p, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        L.ref_write_pbm.restype = C.c_int64
        L.ref_write_pbm.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int, C.c_char_p, C.c_int64]
        L.ref_time_batch.restype = C.c_double
        L.ref_time_batch.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int, C.c_int,
                                     C.POINTER(C.c_int64)]
        _ref = L
    return _ref


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------ generators
def generate(w: int, h: int, density: float, g: int, seed: int) -> np.ndarray:
    """generator.hpp:46-83 -- uint8 [h, w] image of g x g blocks."""
    out = np.empty((h, w), dtype=np.uint8)
    if lib().orc_generate(w, h, float(density), g, seed & (2**64 - 1), _ptr(out)) != 0:
        raise ValueError("generate: invalid spec")
    return out


def generate_rings(w: int, h: int, tile: int = 64, seed: int = 3, salt: float = 0.02) -> np.ndarray:
    out = np.empty((h, w), dtype=np.uint8)
    if lib().orc_generate_rings(w, h, tile, seed, float(salt), _ptr(out)) != 0:
        raise ValueError("generate_rings: invalid spec")
    return out


def cfg4_params(i: int) -> tuple[float, int]:
    d = C.c_double()
    g = C.c_int32()
    lib().orc_cfg4_params(i, C.byref(d), C.byref(g))
    return d.value, g.value


def block_draw(seed: int, r: int, c: int) -> int:
    return lib().orc_block_draw(seed, r, c)


# ------------------------------------------------------------------ labeling
def _canonical(L, fn, free, img: np.ndarray, conn: int, want_labels: bool) -> Canonical:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    r = _OrcResult()
    rc = fn(_ptr(img), w, h, conn, int(want_labels), C.byref(r))
    if rc == -2:
        raise OverflowError("feature accumulator overflow")
    if rc != 0:
        raise ValueError("label_canonical failed")
    try:
        return _to_canonical(r, want_labels)
    finally:
        free(C.byref(r))


def label_canonical(img: np.ndarray, conn: int = 0, want_labels: bool = False) -> Canonical:
    """C restatement: both label_image runs + binarize_labels, canonicalised."""
    L = lib()
    return _canonical(L, L.orc_label_canonical, L.orc_result_free, img, conn, want_labels)


def ref_label_canonical(img: np.ndarray, conn: int = 0, want_labels: bool = False) -> Canonical:
    """The reference itself (oracle/_ref), same contract."""
    L = ref()
    return _canonical(L, L.ref_label_canonical, L.ref_result_free, img, conn, want_labels)


def encode_row(row: np.ndarray, use_ref: bool = False) -> tuple[int, np.ndarray, np.ndarray]:
    row = np.ascontiguousarray(row, dtype=np.uint8)
    w = row.shape[0]
    er = np.zeros(w, dtype=np.int32)
    rlc = np.zeros(w + 2, dtype=np.int32)
    fn = ref().ref_encode_row if use_ref else lib().orc_encode_row
    ner = fn(_ptr(row), w, _ptr(er), _ptr(rlc))
    return ner, er, rlc[:ner + 1]


def flood_label(img: np.ndarray, conn: int = 0) -> tuple[int, np.ndarray, np.ndarray]:
    """oracle.hpp:86-124 -- (count, comp[h,w], comp_fg[count])."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    comp = np.empty((h, w), dtype=np.int32)
    cap = w * h + 1
    fg = np.zeros(cap, dtype=np.uint8)
    n = lib().orc_flood_label(_ptr(img), w, h, conn, _ptr(comp), _ptr(fg), None, cap)
    return n, comp, fg[:n]


def bitquad_euler(img: np.ndarray, conn: int = 0) -> int:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    return lib().orc_bitquad_euler(_ptr(img), w, h, conn)


def fill_holes(img: np.ndarray, conn: int = 0) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    out = np.empty_like(img)
    lib().orc_fill_holes(_ptr(img), w, h, conn, _ptr(out))
    return out


def ref_time_batch(imgs: np.ndarray, conn: int = 0, threads: int = 1) -> tuple[float, int]:
    """Wall seconds of the reference path over a [n, h, w] batch (see ref_shim.cpp)."""
    imgs = np.ascontiguousarray(imgs, dtype=np.uint8)
    n, h, w = imgs.shape
    chk = C.c_int64()
    secs = ref().ref_time_batch(_ptr(imgs), w, h, n, conn, threads, C.byref(chk))
    return secs, chk.value


def filter_components(comps: np.ndarray, selected: np.ndarray):
    """C restatement of analysis.hpp:89-125 on a canonical pre-fill table.
    Returns (parent, features, adjacency); raises ValueError if the exterior is selected."""
    comps = np.ascontiguousarray(comps, dtype=COMPONENT_DTYPE)
    sel = np.ascontiguousarray(selected, dtype=np.uint8)
    n = comps.shape[0]
    parent = np.empty(n, dtype=np.uint32)
    feats = np.empty(n, dtype=FEATURE_DTYPE)
    adj = np.empty(n, dtype=np.uint32)
    rc = lib().orc_filter_components(_ptr(comps), n, _ptr(sel), _ptr(parent), _ptr(feats), _ptr(adj))
    if rc == -1:
        raise ValueError("filter_components: predicate must not select the exterior")
    if rc != 0:
        raise RuntimeError(f"orc_filter_components failed ({rc})")
    return parent, feats, adj


def ref_filter_components(img: np.ndarray, selected: np.ndarray, conn: int = 0):
    """The reference's own filter_components on its label_image result, canonical ids."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    sel = np.ascontiguousarray(selected, dtype=np.uint8)
    n = sel.shape[0]
    h, w = img.shape
    parent = np.empty(n, dtype=np.uint32)
    feats = np.empty(n, dtype=FEATURE_DTYPE)
    adj = np.empty(n, dtype=np.uint32)
    rc = ref().ref_filter_components(_ptr(img), w, h, conn, _ptr(sel), n, _ptr(parent), _ptr(feats), _ptr(adj))
    if rc == -1:
        raise ValueError("filter_components: predicate must not select the exterior")
    if rc != 0:
        raise RuntimeError(f"ref_filter_components failed ({rc})")
    return parent, feats, adj


def ref_read_pbm(data: bytes):
    """The reference's read_pbm: (pixels uint8 [h, w], None) or (None, PbmParseError offset)."""
    w, h, off = C.c_int32(0), C.c_int32(0), C.c_int64(-1)
    cap = max(64, len(data) * 8 + 64)
    px = np.zeros(cap, dtype=np.uint8)
    rc = ref().ref_read_pbm(data, len(data), _ptr(px), cap, C.byref(w), C.byref(h), C.byref(off))
    if rc != 0:
        return None, int(off.value)
    return px[: w.value * h.value].reshape(h.value, w.value).copy(), None


def ref_write_pbm(img: np.ndarray, p1: bool = False) -> bytes:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    h, w = img.shape
    n = ref().ref_write_pbm(_ptr(img), w, h, int(p1), None, 0)
    out = C.create_string_buffer(n)
    ref().ref_write_pbm(_ptr(img), w, h, int(p1), out, n)
    return out.raw[:n]
