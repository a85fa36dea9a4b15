"""One image across ranks as horizontal strips, over the C ABI's strip phases.

Each rank holds its strip of rows in device memory.  Only O(width) data crosses ranks: the
strip's components that touch a cut row ("cut classes": first-pixel key, features, foreground
flag) and the two cut rows' class labels.  The phases (include/runlab_gpu.h) are separated by
four collectives, which this module does with torch.distributed (NCCL over NVLink between GPUs;
any backend whose tensors live where the buffers live):

1. all-gather of the per-strip counts (cut classes, components touching no cut, foreground);
2. all-gather of the strips' exchange records (one equal-size record per rank);
3. all-reduce SUM of the link table (canonical id and parent-chain exit of every cut component,
   filled in by the strip that owns it);
4. all-reduce (SUM / MIN / MAX) of the partial post-fill features of the survivors that cross a
   cut.

``label_strip`` is the per-rank entry point.  ``label_strips_in_process`` runs all strips of an
image in one process on one device, phase by phase in lockstep, with the collectives done by
concatenation/reduction of the same records: it is how the strip path is checked against the
single-image result on a one-GPU box (each strip's kernels run on their own; nothing waits on
another strip inside a kernel).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .runlab import LabelingConfig, _raise

TILE_ROWS = 32


def strip_rows(height: int, n_strips: int) -> list[tuple[int, int]]:
    """Rows (y0, h) of n horizontal strips: multiples of the 32-row tile height, the remainder
    spread over the first strips, the last strip takes the image's ragged end."""
    tiles = (height + TILE_ROWS - 1) // TILE_ROWS
    if n_strips < 1 or n_strips > tiles:
        raise ValueError(f"cannot cut {height} rows into {n_strips} strips of whole tile rows")
    base, extra = divmod(tiles, n_strips)
    out, t = [], 0
    for r in range(n_strips):
        nt = base + (1 if r < extra else 0)
        y0 = t * TILE_ROWS
        y1 = min((t + nt) * TILE_ROWS, height)
        out.append((y0, y1 - y0))
        t += nt
    return out


class _DevArray:
    """Zero-copy view of library-owned device memory for torch (CUDA array interface)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _view(ptr: int, n: int, typestr: str):
    import torch
    if n == 0:
        return torch.empty(0, dtype={"<i8": torch.int64, "<i4": torch.int32}[typestr], device="cuda")
    return torch.as_tensor(_DevArray(ptr, n, typestr), device="cuda")


@dataclass
class StripResult:
    comp_lo: int
    comp_hi: int
    n_components: int
    n_fg: int
    n_holes: int
    euler: int
    n_survivors: int
    y0: int
    h: int
    comps: np.ndarray | None = None
    top: np.ndarray | None = None
    filled: np.ndarray | None = None
    filled_image: np.ndarray | None = None
    labels: np.ndarray | None = None


class StripPhases:
    """The per-rank phases over one context (a ``Labeler``)."""

    def __init__(self, labeler):
        self.lab = labeler
        self.L = labeler._L
        self.ctx = labeler.ctx
        self.W = self.H = 0
        self.info = None
        self._host = {}

    def _check(self, rc):
        if rc != N.RL_OK:
            _raise(rc, self.lab._err())

    def local(self, d_ptr: int, W: int, H: int, y0: int, h: int, cfg: LabelingConfig) -> np.ndarray:
        self.W, self.H = W, H
        info = N.RlStripLocalInfo()
        self._check(self.L.rl_strip_local(self.ctx, C.c_void_p(d_ptr), W, H, y0, h, C.byref(cfg.to_c()),
                                          C.byref(info)))
        self.info = info
        return np.array([info.n_classes, info.n_comps, info.n_fg, info.ty0, info.ty1], dtype=np.int64)

    def export_bytes(self, max_classes: int) -> int:
        return int(self.L.rl_strip_export_bytes(self.W, max_classes))

    def export(self, max_classes: int):
        import torch
        buf = torch.empty(self.export_bytes(max_classes), dtype=torch.uint8, device="cuda")
        self._check(self.L.rl_strip_export(self.ctx, max_classes, C.c_void_p(buf.data_ptr())))
        return buf

    def merge(self, gathered, infos: np.ndarray, max_classes: int):
        n = infos.shape[0]
        arr = (N.RlStripLocalInfo * n)()
        for q in range(n):
            arr[q].n_classes, arr[q].n_comps, arr[q].n_fg = (int(v) for v in infos[q, :3])
            arr[q].ty0, arr[q].ty1 = int(infos[q, 3]), int(infos[q, 4])
        lk = N.RlStripLinks()
        self._check(self.L.rl_strip_merge(self.ctx, C.c_void_p(gathered.data_ptr()), n, arr, max_classes,
                                          C.byref(lk)))
        return _view(lk.d_links, int(lk.n), "<i8")

    def resolve(self):
        p = N.RlStripPartials()
        self._check(self.L.rl_strip_resolve(self.ctx, C.byref(p)))
        k = int(p.k)
        return (_view(p.d_sum, 3 * k, "<i8"), _view(p.d_min, 2 * k, "<i4"), _view(p.d_max, 2 * k, "<i4"),
                _view(p.d_count, 1, "<i8"))

    def finish(self) -> N.RlStripResult:
        r = N.RlStripResult()
        self._check(self.L.rl_strip_finish(self.ctx, C.byref(r)))
        return r

    def _pinned(self, name: str, nbytes: int):
        """Pinned host staging buffers, kept across calls (pinning is slow)."""
        import torch
        buf = self._host.get(name)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1) + nbytes // 8, dtype=torch.uint8).pin_memory()
            self._host[name] = buf
        return buf

    def fetch(self, r: N.RlStripResult, want_labels: bool = False) -> StripResult:
        n = int(r.comp_hi - r.comp_lo)
        npx = int(r.h) * self.W
        comps, top, filled = self._pinned("comps", n * 48), self._pinned("top", n * 4), self._pinned("filled", n * 40)
        img = self._pinned("img", npx)
        labels = self._pinned("labels", npx * 4) if want_labels else None
        o = N.RlHostOutputs(img.data_ptr(), labels.data_ptr() if labels is not None else None, comps.data_ptr(),
                            top.data_ptr(), filled.data_ptr(), max(n, 1), None, None, 0, 0, 0, 0, 0)
        self._check(self.L.rl_strip_fetch(self.ctx, C.byref(r), C.byref(o)))
        return StripResult(int(r.comp_lo), int(r.comp_hi), int(r.n_components), int(r.n_fg), int(r.n_holes),
                           int(r.euler), int(r.n_survivors), int(r.y0), int(r.h),
                           comps.numpy()[: n * 48].view(N.COMPONENT_DTYPE),
                           top.numpy()[: n * 4].view(np.uint32),
                           filled.numpy()[: n * 40].view(N.FEATURE_DTYPE),
                           img.numpy()[:npx].reshape(int(r.h), self.W),
                           None if labels is None else labels.numpy()[: npx * 4].view(np.uint32).reshape(int(r.h), self.W))


def _max_classes(infos: np.ndarray) -> int:
    return int(infos[:, 0].max())


class TorchCollectives:
    """The four strip collectives over a torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def gather_infos(self, info: np.ndarray, device) -> np.ndarray:
        import torch
        t = torch.as_tensor(info, dtype=torch.int64, device=device)
        out = torch.empty(self.world * t.numel(), dtype=torch.int64, device=device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy().reshape(self.world, -1)

    @staticmethod
    def _done(t):
        """The strip phases run on the library's own stream: the collective's result must be in
        memory before the next phase is enqueued."""
        import torch
        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()

    def gather_records(self, rec):
        import torch
        out = torch.empty(self.world * rec.numel(), dtype=rec.dtype, device=rec.device)
        self.dist.all_gather_into_tensor(out, rec, group=self.group)
        self._done(out)
        return out

    def reduce_links(self, links):
        if links.numel():
            self.dist.all_reduce(links, op=self.dist.ReduceOp.SUM, group=self.group)
            self._done(links)

    def reduce_partials(self, psum, pmin, pmax, pcnt):
        R = self.dist.ReduceOp
        for t, op in ((psum, R.SUM), (pmin, R.MIN), (pmax, R.MAX), (pcnt, R.SUM)):
            if t.numel():
                self.dist.all_reduce(t, op=op, group=self.group)
        self._done(pcnt)


class HostStagedCollectives(TorchCollectives):
    """The same four collectives over a CPU backend (gloo): device tensors are staged through
    host memory around each collective.  For process groups without NCCL -- e.g. ranks that
    share one GPU, where NCCL refuses duplicate devices."""

    def gather_infos(self, info: np.ndarray, device) -> np.ndarray:
        return super().gather_infos(info, "cpu")

    def gather_records(self, rec):
        out = super().gather_records(rec.cpu())
        return out.to(rec.device)

    def reduce_links(self, links):
        h = links.cpu()
        super().reduce_links(h)
        links.copy_(h)
        self._done(links)

    def reduce_partials(self, psum, pmin, pmax, pcnt):
        hs = [t.cpu() for t in (psum, pmin, pmax, pcnt)]
        super().reduce_partials(*hs)
        for d, h in zip((psum, pmin, pmax, pcnt), hs):
            d.copy_(h)
        self._done(pcnt)


_PHASES: dict[int, StripPhases] = {}


def label_strip(labeler, d_strip_ptr: int, W: int, H: int, y0: int, h: int, config: LabelingConfig,
                coll: TorchCollectives, fetch: bool = True) -> StripResult:
    """This rank's strip of one W x H image (rows [y0, y0 + h) at d_strip_ptr).  With fetch the
    returned arrays are views of pinned staging buffers reused by the next call on this context."""
    ph = _PHASES.get(id(labeler))
    if ph is None or ph.lab is not labeler:
        ph = _PHASES[id(labeler)] = StripPhases(labeler)
    infos = coll.gather_infos(ph.local(d_strip_ptr, W, H, y0, h, config), "cuda")
    mc = _max_classes(infos)
    gathered = coll.gather_records(ph.export(mc))
    coll.reduce_links(ph.merge(gathered, infos, mc))
    psum, pmin, pmax, pcnt = ph.resolve()
    coll.reduce_partials(psum, pmin, pmax, pcnt)
    r = ph.finish()
    if not fetch:
        return StripResult(int(r.comp_lo), int(r.comp_hi), int(r.n_components), int(r.n_fg), int(r.n_holes),
                           int(r.euler), int(r.n_survivors), int(r.y0), int(r.h))
    return ph.fetch(r, config.relabel)


def label_strips_in_process(labelers, d_strip_ptrs, W: int, H: int, rows, config: LabelingConfig):
    """All strips of one image in this process (one context per strip), phases in lockstep."""
    import torch
    phs = [StripPhases(lab) for lab in labelers]
    infos = np.stack([ph.local(p, W, H, y0, h, config) for ph, p, (y0, h) in zip(phs, d_strip_ptrs, rows)])
    mc = _max_classes(infos)
    gathered = torch.cat([ph.export(mc) for ph in phs])
    torch.cuda.synchronize()
    links = [ph.merge(gathered, infos, mc) for ph in phs]
    tot = torch.stack(links).sum(dim=0)
    for lk in links:
        lk.copy_(tot)
    torch.cuda.synchronize()
    parts = [ph.resolve() for ph in phs]
    for j, red in enumerate((torch.sum, torch.amin, torch.amax, torch.sum)):
        if parts[0][j].numel():
            stacked = torch.stack([p[j] for p in parts])
            tot = red(stacked, dim=0)
            for p in parts:
                p[j].copy_(tot)
    torch.cuda.synchronize()
    out = []
    for ph in phs:  # copies: the staging buffers are per context
        r = ph.fetch(ph.finish(), config.relabel)
        for f in ("comps", "top", "filled", "filled_image", "labels"):
            v = getattr(r, f)
            setattr(r, f, None if v is None else v.copy())
        out.append(r)
    return out


def label_strips_native(labelers, d_strip_ptrs, W: int, H: int, config: LabelingConfig,
                        fetch: bool = True) -> list[StripResult]:
    """All strips of one image through the library's single-call driver (rl_label_strips): one
    context per strip -- one per GPU of the node, or several on one GPU -- with the collectives
    done as device-to-device copies (peer access over NVLink) and reduction kernels, the strips'
    phases on one host thread each.  Rows per strip: strip_rows(H, len(labelers))."""
    k = len(labelers)
    L = labelers[0]._L
    ctxs = (C.c_void_p * k)(*[lab.ctx for lab in labelers])
    ptrs = (C.c_void_p * k)(*d_strip_ptrs)
    res = (N.RlStripResult * k)()
    rc = L.rl_label_strips(ctxs, k, ptrs, W, H, C.byref(config.to_c()), res)
    if rc != N.RL_OK:
        _raise(rc, labelers[0]._err())
    out = []
    for lab, r in zip(labelers, res):
        ph = _PHASES.get(id(lab))
        if ph is None or ph.lab is not lab:
            ph = _PHASES[id(lab)] = StripPhases(lab)
        ph.W, ph.H = W, H
        if not fetch:
            out.append(StripResult(int(r.comp_lo), int(r.comp_hi), int(r.n_components), int(r.n_fg),
                                   int(r.n_holes), int(r.euler), int(r.n_survivors), int(r.y0), int(r.h)))
            continue
        sr = ph.fetch(r, config.relabel)
        for f in ("comps", "top", "filled", "filled_image", "labels"):  # the staging is per context
            v = getattr(sr, f)
            setattr(sr, f, None if v is None else v.copy())
        out.append(sr)
    return out


def concat(results: list[StripResult]) -> dict:
    """Whole-image tables from the strips' owned ranges (comparable with a single-image call)."""
    rs = sorted(results, key=lambda r: r.y0)
    d = dict(n_components=rs[0].n_components, n_fg=rs[0].n_fg, n_holes=rs[0].n_holes, euler=rs[0].euler,
             n_survivors=rs[0].n_survivors,
             comps=np.concatenate([r.comps for r in rs]), top=np.concatenate([r.top for r in rs]),
             filled=np.concatenate([r.filled for r in rs]),
             filled_image=np.concatenate([r.filled_image for r in rs], axis=0))
    if rs[0].labels is not None:
        d["labels"] = np.concatenate([r.labels for r in rs], axis=0)
    return d
