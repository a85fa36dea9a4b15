"""Python mirror of the reference's labeling/analysis interface, backed by the sm_100a path.

Same names, argument meaning and error behaviour as the reference C++ API (paths relative to
``/root/reference/proj/include/runlab/``):

=========================  ==========================================================
``Connectivity``            ``types.hpp:18-21``
``LabelingConfig``          ``labeling.hpp:20-27``
``LabelingResult``          ``labeling.hpp:29-50`` (+ ``EquivalenceTable`` tables.hpp:37-84,
                            ``AdjacencyTable`` tables.hpp:94-108)
``label_image``             ``labeling.hpp:336-339``
``timed_label_image``       ``labeling.hpp:343-348`` (device phase times, ``StepTimes``)
``binarize_labels``         ``labeling.hpp:354-360``
``components`` / ``holes``  ``analysis.hpp:23-53``
``adjacency_tree``          ``analysis.hpp:56-71``
``euler_number``            ``analysis.hpp:75-79``
=========================  ==========================================================

Labels are the canonical ids (raster order of each component's first pixel, exterior 0),
which equal the reference's root labels renumbered in ascending order; the reference's raw
provisional labels are a by-product of its sequential scan and are not reproduced.  Errors:
``ValueError`` = std::invalid_argument, ``LogicError`` = std::logic_error,
``OverflowError`` = std::overflow_error.

Batches of equally-sized images go through ``Labeler.label_batch`` (one pipeline over all
tiles of all images).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

NO_LABEL = 0xFFFFFFFF


class LogicError(RuntimeError):
    """std::logic_error"""


class Connectivity(enum.IntEnum):
    fg8_bg4 = 0
    fg4_bg8 = 1


@dataclass
class LabelingConfig:
    connectivity: Connectivity = Connectivity.fg8_bg4
    fill_holes: bool = False
    compute_features: bool = False
    relabel: bool = False
    densify_labels: bool = False
    compute_euler: bool = False

    def to_c(self) -> N.RlConfig:
        return N.RlConfig(int(self.connectivity), int(self.fill_holes), int(self.compute_features),
                          int(self.relabel), int(self.densify_labels), int(self.compute_euler))


@dataclass
class StepTimes:
    """Device phase times in ms (CUDA events), cf. labeling.hpp:253-259."""
    analyze_ms: float = 0.0
    merge_ms: float = 0.0
    emit_ms: float = 0.0
    total_ms: float = 0.0
    relabel_ms: float = 0.0  # densified label ids / survivor compaction after the emit pass


@dataclass
class EquivalenceTable:
    t: np.ndarray       # uint32 parent per label (T[e] <= e)
    parity: np.ndarray  # uint8, 1 = foreground

    def size(self) -> int:
        return int(self.t.shape[0])

    def parent(self, e: int) -> int:
        return int(self.t[e])

    def is_root(self, e: int) -> bool:
        return int(self.t[e]) == e

    def is_foreground(self, e: int) -> bool:
        return bool(self.parity[e])

    def find(self, e: int) -> int:
        while int(self.t[e]) != e:
            e = int(self.t[e])
        return e


@dataclass
class LabelingResult:
    width: int
    height: int
    config: LabelingConfig
    equivalences: EquivalenceTable
    adjacency: np.ndarray                 # uint32; adjacency[0] = NO_LABEL
    features: np.ndarray | None = None    # FEATURE_DTYPE per label
    labels: np.ndarray | None = None      # uint32 [h, w]
    fg_count: int | None = None
    hole_count: int | None = None
    euler: int | None = None
    times: StepTimes = field(default_factory=StepTimes)

    def roots(self) -> list[int]:
        t = self.equivalences.t
        return [int(e) for e in np.nonzero(t == np.arange(t.shape[0], dtype=t.dtype))[0]]


@dataclass
class BatchResult:
    """Canonical per-image tables of one batch call (the C ABI's rl_result)."""
    width: int
    height: int
    n_images: int
    n_components: np.ndarray
    n_fg: np.ndarray
    n_holes: np.ndarray
    euler: np.ndarray
    n_survivors: np.ndarray
    comp_offset: np.ndarray
    comps: np.ndarray          # COMPONENT_DTYPE, all images concatenated
    top: np.ndarray
    filled: np.ndarray
    filled_image: np.ndarray   # uint8 [n, h, w]
    labels: np.ndarray | None  # uint32 [n, h, w]
    times: StepTimes

    def image(self, i: int) -> dict:
        a, b = int(self.comp_offset[i]), int(self.comp_offset[i + 1])
        return dict(n_components=int(self.n_components[i]), n_fg=int(self.n_fg[i]),
                    n_holes=int(self.n_holes[i]), euler=int(self.euler[i]),
                    n_survivors=int(self.n_survivors[i]), comps=self.comps[a:b],
                    top=self.top[a:b], filled=self.filled[a:b],
                    filled_image=self.filled_image[i],
                    labels=None if self.labels is None else self.labels[i])


class PbmParseError(ValueError):
    """runlab::PbmParseError (io.hpp:16-23): malformed PBM input at `byte_offset`."""

    def __init__(self, msg: str, byte_offset: int):
        super().__init__(msg)
        self.byte_offset = byte_offset


def read_pbm_header(data: bytes) -> N.RlPbmInfo:
    """Header of a P1/P4 file with the reference's rules (raises PbmParseError)."""
    info = N.RlPbmInfo()
    buf = C.create_string_buffer(bytes(data), len(data))
    rc = N.load().rl_pbm_parse(buf, len(data), C.byref(info))
    if rc == N.RL_EFORMAT:
        raise PbmParseError(info.message.decode(), int(info.error_offset))
    if rc != N.RL_OK:
        _raise(rc, "rl_pbm_parse failed")
    return info


def pack_p4(img: np.ndarray) -> np.ndarray:
    """uint8 [..., h, w] 0/1 pixels -> P4 rows [..., h, ceil(w/8)] (MSB-first, zero pad bits)."""
    return np.packbits(np.asarray(img, dtype=np.uint8) & 1, axis=-1)


def unpack_p4(rows: np.ndarray, w: int) -> np.ndarray:
    return np.unpackbits(rows, axis=-1)[..., :w]


def _raise(code: int, msg: str):
    if code == N.RL_EINVAL:
        raise ValueError(msg)
    if code == N.RL_ELOGIC:
        raise LogicError(msg)
    if code == N.RL_EOVERFLOW:
        raise OverflowError(msg)
    if code == N.RL_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


class Labeler:
    """One C-ABI context (device, stream, workspace).  One per thread."""

    def __init__(self, device: int = 0):
        self._L = N.load()
        self._ctx = self._L.rl_create(device)
        if not self._ctx:
            raise RuntimeError("rl_create failed: no usable CUDA device (no CPU fallback)")

    def close(self):
        if getattr(self, "_ctx", None):
            self._L.rl_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ctx(self):
        return self._ctx

    def _err(self) -> str:
        m = self._L.rl_last_error(self._ctx)
        return m.decode() if m else ""

    def label_batch(self, images: np.ndarray, config: LabelingConfig | None = None) -> BatchResult:
        """images: uint8 [n, h, w] (or [h, w]) host array with 0/1 pixels."""
        config = config or LabelingConfig()
        imgs = np.ascontiguousarray(images, dtype=np.uint8)
        if imgs.ndim == 2:
            imgs = imgs[None]
        if imgs.ndim != 3:
            raise ValueError("images must be [n, h, w]")
        n, h, w = imgs.shape
        cfg = config.to_c()
        res = N.RlResult()
        rc = self._L.rl_label(self._ctx, imgs.ctypes.data_as(C.c_void_p), w, h, n, C.byref(cfg),
                              C.byref(res))
        if rc != N.RL_OK:
            _raise(rc, self._err())
        try:
            return self._to_batch(res)
        finally:
            self._L.rl_result_free(C.byref(res))

    def label_device(self, d_ptr: int, w: int, h: int, n: int, config: LabelingConfig,
                     stream: int | None = None, pixel_format: int = N.RL_PIXELS_U8):
        """Enqueue the pipeline on a device-resident batch (no host copies, no sync)."""
        if stream is not None:
            self._L.rl_set_stream(self._ctx, C.c_void_p(stream))
        cfg = config.to_c()
        rc = self._L.rl_label_device_fmt(self._ctx, C.c_void_p(d_ptr), w, h, n, C.byref(cfg), pixel_format)
        if rc != N.RL_OK:
            _raise(rc, self._err())

    def sync(self):
        rc = self._L.rl_sync(self._ctx)
        if rc != N.RL_OK:
            _raise(rc, self._err())

    def fetch(self) -> BatchResult:
        res = N.RlResult()
        rc = self._L.rl_fetch(self._ctx, C.byref(res))
        if rc != N.RL_OK:
            _raise(rc, self._err())
        try:
            return self._to_batch(res)
        finally:
            self._L.rl_result_free(C.byref(res))

    def label_into(self, pixels_ptr: int, w: int, h: int, n: int, config: LabelingConfig,
                   outs: N.RlHostOutputs, pixel_format: int = N.RL_PIXELS_U8) -> N.RlHostOutputs:
        """rl_label_into: host pixels in, caller-owned host outputs (the e2e entry point)."""
        cfg = config.to_c()
        rc = self._L.rl_label_into_fmt(self._ctx, C.c_void_p(pixels_ptr), w, h, n, C.byref(cfg), pixel_format,
                                       C.byref(outs))
        if rc != N.RL_OK:
            _raise(rc, self._err())
        return outs

    def fill_pbm(self, data: bytes, config: LabelingConfig | None = None) -> bytes:
        """`runlab fill`: PBM (P1/P4) bytes in, the hole-filled image as a P4 file out."""
        config = config or LabelingConfig(fill_holes=True)
        info = read_pbm_header(data)
        cap = 64 + ((info.width + 7) // 8) * info.height
        out = C.create_string_buffer(cap)
        n = C.c_size_t(0)
        src = C.create_string_buffer(bytes(data), len(data))
        rc = self._L.rl_fill_pbm(self._ctx, src, len(data), C.byref(config.to_c()), out, cap, C.byref(n), None,
                                 C.byref(info))
        if rc == N.RL_EFORMAT:
            raise PbmParseError(info.message.decode(), int(info.error_offset))
        if rc != N.RL_OK:
            _raise(rc, self._err())
        return out.raw[: n.value]

    def phase_times(self, back: int = 0) -> StepTimes:
        t = N.RlTimes()
        rc = self._L.rl_phase_times(self._ctx, back, C.byref(t))
        if rc != N.RL_OK:
            _raise(rc, "phase times unavailable")
        return StepTimes(t.analyze_ms, t.merge_ms, t.emit_ms, t.total_ms, t.relabel_ms)

    def stream(self) -> int:
        return int(self._L.rl_stream(self._ctx) or 0)

    def set_pipelines(self, k: int) -> None:
        """Concurrent pipelines for large device batches (rl_set_pipelines); 1 = one pipeline."""
        if self._L.rl_set_pipelines(self._ctx, int(k)) != N.RL_OK:
            _raise(N.RL_EINVAL, "pipelines must be >= 1")

    def workspace_bytes(self) -> int:
        """Device bytes held by this context's grow-only tables."""
        return int(self._L.rl_workspace_bytes(self._ctx))

    def launch_count(self) -> int:
        return int(self._L.rl_last_launch_count(self._ctx))

    def used_graph(self) -> bool:
        return bool(self._L.rl_last_used_graph(self._ctx))

    def device_filled_image(self) -> int:
        return int(self._L.rl_device_filled_image(self._ctx) or 0)

    @staticmethod
    def _to_batch(res: N.RlResult) -> BatchResult:
        n, h, w = res.n_images, res.height, res.width
        off = N.copy_out(res.comp_offset, np.int64, n + 1)
        total = int(off[-1])
        labels = None
        if res.labels:
            labels = N.copy_out(res.labels, np.uint32, n * h * w).reshape(n, h, w)
        return BatchResult(
            width=w, height=h, n_images=n,
            n_components=N.copy_out(res.n_components, np.int64, n),
            n_fg=N.copy_out(res.n_fg, np.int64, n),
            n_holes=N.copy_out(res.n_holes, np.int64, n),
            euler=N.copy_out(res.euler, np.int64, n),
            n_survivors=N.copy_out(res.n_survivors, np.int64, n),
            comp_offset=off,
            comps=N.copy_out(res.comps, N.COMPONENT_DTYPE, total),
            top=N.copy_out(res.top, np.uint32, total),
            filled=N.copy_out(res.filled, N.FEATURE_DTYPE, total),
            filled_image=N.copy_out(res.filled_image, np.uint8, n * h * w).reshape(n, h, w),
            labels=labels,
            times=StepTimes(res.times.analyze_ms, res.times.merge_ms, res.times.emit_ms,
                            res.times.total_ms, res.times.relabel_ms))


_default: Labeler | None = None


def default_labeler() -> Labeler:
    global _default
    if _default is None:
        _default = Labeler(0)
    return _default


def _empty_features(n: int) -> np.ndarray:
    f = np.zeros(n, dtype=N.FEATURE_DTYPE)
    f["row_min"] = np.iinfo(np.int32).max
    f["col_min"] = np.iinfo(np.int32).max
    f["row_max"] = np.iinfo(np.int32).min
    f["col_max"] = np.iinfo(np.int32).min
    return f


def _result_from(b: BatchResult, i: int, config: LabelingConfig) -> LabelingResult:
    im = b.image(i)
    comps, top = im["comps"], im["top"]
    n = comps.shape[0]
    ids = np.arange(n, dtype=np.uint32)
    parity = (comps["flags"] & 1).astype(np.uint8)
    t = top.copy() if config.fill_holes else ids.copy()
    adj = comps["parent"].astype(np.uint32)
    adj[0] = NO_LABEL
    feats = None
    if config.compute_features:
        feats = np.empty(n, dtype=N.FEATURE_DTYPE)
        for k in N.FEATURE_DTYPE.names:
            feats[k] = comps[k]
        if config.fill_holes:
            surv = top == ids
            feats[surv] = im["filled"][surv]
    res = LabelingResult(width=b.width, height=b.height, config=config,
                         equivalences=EquivalenceTable(t=t, parity=parity), adjacency=adj,
                         features=feats, labels=im["labels"].copy() if im["labels"] is not None else None,
                         times=b.times)
    if config.compute_euler:
        res.fg_count, res.hole_count, res.euler = im["n_fg"], im["n_holes"], im["euler"]
    return res


def label_image(image: np.ndarray, config: LabelingConfig | None = None,
                labeler: Labeler | None = None) -> LabelingResult:
    """labeling.hpp:336-339 -- FG/BG labeling + analysis of one binary image on the GPU."""
    config = config or LabelingConfig()
    if config.densify_labels and not config.relabel:
        raise ValueError("label_image: densify_labels requires relabel")
    img = np.asarray(image, dtype=np.uint8)
    if img.ndim != 2 or img.shape[0] < 1 or img.shape[1] < 1:
        raise ValueError("image must be a non-empty 2-D array")
    b = (labeler or default_labeler()).label_batch(img[None], config)
    return _result_from(b, 0, config)


def timed_label_image(image: np.ndarray, config: LabelingConfig,
                      labeler: Labeler | None = None) -> tuple[LabelingResult, StepTimes]:
    """labeling.hpp:343-348 -- same result, plus per-phase device times."""
    res = label_image(image, config, labeler)
    return res, res.times


def binarize_labels(labels: np.ndarray, eq: EquivalenceTable) -> np.ndarray:
    """labeling.hpp:354-360 -- pixel is foreground iff its label's parity is."""
    return eq.parity[np.asarray(labels, dtype=np.int64)].astype(np.uint8)


@dataclass
class ComponentRecord:
    root: int
    foreground: bool
    parent_root: int
    depth: int
    features: np.void | None


def components(res: LabelingResult) -> list[ComponentRecord]:
    """analysis.hpp:23-41 -- one record per surviving root, ascending."""
    out = []
    t = res.equivalences.t
    depth = np.zeros(t.shape[0], dtype=np.int32)
    for e in range(t.shape[0]):
        if int(t[e]) != e:
            continue
        parent = NO_LABEL
        if e != 0:
            parent = int(res.adjacency[e])
            depth[e] = depth[parent] + 1
        feat = res.features[e] if res.features is not None else _empty_features(1)[0]
        out.append(ComponentRecord(e, bool(res.equivalences.parity[e]), parent, int(depth[e]), feat))
    return out


def holes(res: LabelingResult) -> list[ComponentRecord]:
    """analysis.hpp:46-53"""
    if res.config.fill_holes:
        raise LogicError("holes: result was computed with hole filling")
    return [r for r in components(res) if not r.foreground and r.root != 0]


@dataclass
class ComponentTree:
    nodes: list[ComponentRecord]
    children: list[list[int]]


def adjacency_tree(res: LabelingResult) -> ComponentTree:
    """analysis.hpp:56-71"""
    nodes = components(res)
    index = {n.root: i for i, n in enumerate(nodes)}
    children: list[list[int]] = [[] for _ in nodes]
    for i in range(1, len(nodes)):
        children[index[nodes[i].parent_root]].append(i)
    return ComponentTree(nodes, children)


def euler_number(res: LabelingResult) -> int:
    """analysis.hpp:75-79"""
    if res.euler is None:
        raise LogicError("euler_number: labeling ran without compute_euler")
    return int(res.euler)


# ---------------------------------------------------------------------------------------
# device-side input generators (generator.hpp:46-83 and the BASELINE configs)
# ---------------------------------------------------------------------------------------
def generate_device(d_ptr: int, w: int, h: int, density: float, g: int, seed: int,
                    stream: int | None = None) -> None:
    """generate() on the device into w*h bytes at d_ptr (bit-identical to the reference)."""
    rc = N.load().rl_generate(C.c_void_p(stream or 0), C.c_void_p(d_ptr), w, h, float(density), g,
                              seed & (2**64 - 1))
    if rc != N.RL_OK:
        _raise(rc, "generate: invalid spec" if rc == N.RL_EINVAL else "generate failed")


def filter_components(comps, selected, stream: int | None = None):
    """analysis.hpp:89-125 on one image's canonical component table (COMPONENT_DTYPE records,
    host numpy or a CUDA uint8 tensor of n*48 bytes) with a selection mask (one flag per
    component; the reference's predicate evaluated by the caller).  Returns host arrays
    (parent, features, adjacency) -- see rl_filter_components.  ValueError if the exterior is
    selected (std::invalid_argument in the reference)."""
    import torch
    if isinstance(comps, np.ndarray):
        comps = np.ascontiguousarray(comps, dtype=N.COMPONENT_DTYPE)
        n = comps.shape[0]
        d_comps = torch.from_numpy(comps.view(np.uint8).reshape(-1)).cuda()
    else:
        d_comps = comps
        n = d_comps.numel() // 48
    sel = selected if isinstance(selected, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(selected, dtype=np.uint8))
    d_sel = sel.to(device=d_comps.device, dtype=torch.uint8).contiguous()
    if d_sel.numel() != n:
        raise ValueError("selected must have one flag per component")
    d_parent = torch.empty(n, dtype=torch.int32, device=d_comps.device)
    d_feat = torch.empty(n * 40, dtype=torch.uint8, device=d_comps.device)
    d_adj = torch.empty(n, dtype=torch.int32, device=d_comps.device)
    if stream is None:
        stream = torch.cuda.current_stream(d_comps.device).cuda_stream
    rc = N.load().rl_filter_components(C.c_void_p(stream), C.c_void_p(d_comps.data_ptr()), n,
                                       C.c_void_p(d_sel.data_ptr()), C.c_void_p(d_parent.data_ptr()),
                                       C.c_void_p(d_feat.data_ptr()), C.c_void_p(d_adj.data_ptr()))
    if rc == N.RL_EINVAL:
        raise ValueError("filter_components: predicate must not select the exterior")
    if rc != N.RL_OK:
        _raise(rc, "rl_filter_components failed")
    return (d_parent.cpu().numpy().view(np.uint32), d_feat.cpu().numpy().view(N.FEATURE_DTYPE),
            d_adj.cpu().numpy().view(np.uint32))


def generate_rows_device(d_ptr: int, w: int, h: int, y0: int, rows: int, density: float, g: int, seed: int,
                         stream: int | None = None) -> None:
    """Rows [y0, y0 + rows) of generate(w, h, density, g, seed) on the device (one strip)."""
    rc = N.load().rl_generate_rows(C.c_void_p(stream or 0), C.c_void_p(d_ptr), w, h, y0, rows, float(density),
                                   g, seed)
    if rc != N.RL_OK:
        raise ValueError("rl_generate_rows: invalid arguments")


def generate_rings_device(d_ptr: int, w: int, h: int, tile: int = 64, seed: int = 3,
                          salt: float = 0.02, stream: int | None = None) -> None:
    """Config-3 nested-ring image on the device."""
    rc = N.load().rl_generate_rings(C.c_void_p(stream or 0), C.c_void_p(d_ptr), w, h, tile, seed,
                                    float(salt))
    if rc != N.RL_OK:
        _raise(rc, "generate_rings failed")


def cfg4_params(i: int) -> tuple[float, int]:
    d = C.c_double()
    g = C.c_int32()
    N.load().rl_cfg4_params(i, C.byref(d), C.byref(g))
    return d.value, g.value


def cfg2_cells() -> list[tuple[float, int]]:
    """BASELINE config 2: density k/20 (k = 0..20) x granularity {1,2,4,8,16}."""
    return [(k / 20.0, g) for k in range(21) for g in (1, 2, 4, 8, 16)]
