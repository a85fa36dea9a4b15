"""ctypes binding of the C ABI in ``include/runlab_gpu.h`` (``librunlab_gpu.so``).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).  There is no
CPU fallback: if the library or a GPU is missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RUNLAB_GPU_LIB", os.path.join(HERE, "librunlab_gpu.so"))

RL_OK, RL_EINVAL, RL_ELOGIC, RL_EOVERFLOW, RL_ECUDA, RL_ENOMEM, RL_EINTERNAL, RL_ENOSPC, RL_EFORMAT = range(9)
RL_PIXELS_U8, RL_PIXELS_P4 = 0, 1

EXPORTED_SYMBOLS = (
    "rl_create", "rl_destroy", "rl_last_error", "rl_label", "rl_result_free", "rl_label_device",
    "rl_sync", "rl_fetch", "rl_device_filled_image", "rl_device_labels", "rl_device_comps",
    "rl_stream", "rl_set_stream", "rl_last_launch_count", "rl_tile_shape", "rl_label_into",
    "rl_phase_times", "rl_generate", "rl_generate_rings", "rl_cfg4_params", "rl_last_used_graph",
    "rl_strip_local", "rl_strip_export_bytes", "rl_strip_export", "rl_strip_merge", "rl_strip_resolve",
    "rl_strip_finish",
    "rl_strip_fetch", "rl_strip_rows", "rl_label_strips", "rl_label_strips_host", "rl_generate_rows", "rl_filter_components",
    "rl_filter_components_host", "rl_label_device_fmt", "rl_label_into_fmt", "rl_pbm_parse", "rl_pbm_p1_to_p4",
    "rl_pbm_p4_header", "rl_fill_pbm", "rl_generate_host", "rl_workspace_bytes", "rl_set_pipelines",
)

FEATURE_DTYPE = np.dtype([("s", "<i8"), ("sx", "<i8"), ("sy", "<i8"), ("row_min", "<i4"),
                          ("row_max", "<i4"), ("col_min", "<i4"), ("col_max", "<i4")])
COMPONENT_DTYPE = np.dtype([("s", "<i8"), ("sx", "<i8"), ("sy", "<i8"), ("row_min", "<i4"),
                            ("row_max", "<i4"), ("col_min", "<i4"), ("col_max", "<i4"),
                            ("parent", "<u4"), ("flags", "<u4")])


class RlConfig(C.Structure):
    _fields_ = [("connectivity", C.c_int32), ("fill_holes", C.c_int32),
                ("compute_features", C.c_int32), ("relabel", C.c_int32),
                ("densify_labels", C.c_int32), ("compute_euler", C.c_int32)]


class RlTimes(C.Structure):
    _fields_ = [("analyze_ms", C.c_float), ("merge_ms", C.c_float), ("emit_ms", C.c_float),
                ("total_ms", C.c_float), ("relabel_ms", C.c_float)]


class RlResult(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("n_images", C.c_int32),
                ("n_components", C.c_void_p), ("n_fg", C.c_void_p), ("n_holes", C.c_void_p),
                ("euler", C.c_void_p), ("n_survivors", C.c_void_p), ("comp_offset", C.c_void_p),
                ("comps", C.c_void_p), ("top", C.c_void_p), ("filled", C.c_void_p),
                ("filled_image", C.c_void_p), ("labels", C.c_void_p), ("times", RlTimes)]


class RlHostOutputs(C.Structure):
    _fields_ = [("filled_image", C.c_void_p), ("labels", C.c_void_p), ("comps", C.c_void_p),
                ("top", C.c_void_p), ("filled", C.c_void_p), ("comp_capacity", C.c_int64),
                ("summary", C.c_void_p), ("comp_offset", C.c_void_p), ("comps_needed", C.c_int64),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("filled_layout", C.c_int32),
                ("reserved", C.c_int32)]


class RlPbmInfo(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("format", C.c_int32), ("pad", C.c_int32),
                ("raster_offset", C.c_int64), ("error_offset", C.c_int64), ("message", C.c_char * 96)]


class RlStripLocalInfo(C.Structure):
    _fields_ = [("n_classes", C.c_int64), ("n_comps", C.c_int64), ("n_fg", C.c_int64), ("ty0", C.c_int32),
                ("ty1", C.c_int32), ("status", C.c_int32), ("pad", C.c_int32)]


class RlStripLinks(C.Structure):
    _fields_ = [("d_links", C.c_void_p), ("n", C.c_int64)]


class RlStripPartials(C.Structure):
    _fields_ = [("d_sum", C.c_void_p), ("d_min", C.c_void_p), ("d_max", C.c_void_p),
                ("d_count", C.c_void_p), ("k", C.c_int64)]


class RlStripResult(C.Structure):
    _fields_ = [("comp_lo", C.c_int64), ("comp_hi", C.c_int64), ("n_components", C.c_int64),
                ("n_fg", C.c_int64), ("n_holes", C.c_int64), ("euler", C.c_int64),
                ("n_survivors", C.c_int64), ("y0", C.c_int32), ("h", C.c_int32)]


_lib = None


def load() -> C.CDLL:
    """Load librunlab_gpu.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() first "
                           "(the CUDA path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.rl_create.restype = C.c_void_p
    L.rl_create.argtypes = [C.c_int]
    L.rl_destroy.argtypes = [C.c_void_p]
    L.rl_last_error.restype = C.c_char_p
    L.rl_last_error.argtypes = [C.c_void_p]
    L.rl_label.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                           C.POINTER(RlConfig), C.POINTER(RlResult)]
    L.rl_result_free.argtypes = [C.POINTER(RlResult)]
    L.rl_label_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                  C.POINTER(RlConfig)]
    L.rl_sync.argtypes = [C.c_void_p]
    L.rl_fetch.argtypes = [C.c_void_p, C.POINTER(RlResult)]
    for name in ("rl_device_filled_image", "rl_device_labels", "rl_device_comps", "rl_stream"):
        getattr(L, name).restype = C.c_void_p
        getattr(L, name).argtypes = [C.c_void_p]
    L.rl_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    L.rl_last_launch_count.argtypes = [C.c_void_p]
    L.rl_set_pipelines.argtypes = [C.c_void_p, C.c_int]
    L.rl_workspace_bytes.restype = C.c_int64
    L.rl_workspace_bytes.argtypes = [C.c_void_p]
    L.rl_last_used_graph.argtypes = [C.c_void_p]
    L.rl_tile_shape.argtypes = [C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.rl_label_into.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                C.POINTER(RlConfig), C.POINTER(RlHostOutputs)]
    L.rl_phase_times.argtypes = [C.c_void_p, C.c_int, C.POINTER(RlTimes)]
    L.rl_generate.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                              C.c_uint64]
    L.rl_filter_components.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
    L.rl_label_device_fmt.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                      C.POINTER(RlConfig), C.c_int32]
    L.rl_label_into_fmt.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                    C.POINTER(RlConfig), C.c_int32, C.POINTER(RlHostOutputs)]
    L.rl_pbm_parse.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(RlPbmInfo)]
    L.rl_pbm_p1_to_p4.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(RlPbmInfo), C.c_void_p]
    L.rl_pbm_p4_header.restype = C.c_size_t
    L.rl_pbm_p4_header.argtypes = [C.c_int32, C.c_int32, C.c_char_p, C.c_size_t]
    L.rl_fill_pbm.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(RlConfig), C.c_void_p, C.c_size_t,
                              C.POINTER(C.c_size_t), C.POINTER(RlHostOutputs), C.POINTER(RlPbmInfo)]
    L.rl_generate_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                   C.c_double, C.c_int32, C.c_uint64]
    L.rl_generate_rings.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_uint64, C.c_double]
    L.rl_cfg4_params.argtypes = [C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_int32)]
    L.rl_strip_local.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                 C.POINTER(RlConfig), C.POINTER(RlStripLocalInfo)]
    L.rl_strip_export_bytes.restype = C.c_int64
    L.rl_strip_export_bytes.argtypes = [C.c_int32, C.c_int64]
    L.rl_strip_export.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
    L.rl_strip_merge.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(RlStripLocalInfo),
                                 C.c_int64, C.POINTER(RlStripLinks)]
    L.rl_strip_resolve.argtypes = [C.c_void_p, C.POINTER(RlStripPartials)]
    L.rl_strip_finish.argtypes = [C.c_void_p, C.POINTER(RlStripResult)]
    L.rl_strip_fetch.argtypes = [C.c_void_p, C.POINTER(RlStripResult), C.POINTER(RlHostOutputs)]
    L.rl_strip_rows.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.rl_label_strips.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(C.c_void_p), C.c_int32, C.c_int32,
                                  C.POINTER(RlConfig), C.POINTER(RlStripResult)]
    L.rl_label_strips_host.argtypes = [C.POINTER(C.c_void_p), C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                                       C.POINTER(RlConfig), C.POINTER(RlStripResult)]
    _lib = L
    return L


def copy_out(ptr: int, dtype, n: int) -> np.ndarray:
    dtype = np.dtype(dtype)
    if n == 0 or not ptr:
        return np.zeros(n, dtype=dtype)
    buf = (C.c_char * (n * dtype.itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype).copy()
