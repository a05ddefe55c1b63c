"""ctypes binding of the C ABI in include/hashpoint_b200.h (libhp_b200.so).

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, every compute entry point raises RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HP_LIB: an alternative build of the same ABI (A/B measurements only)
LIB_PATH = os.environ.get("HP_LIB") or os.path.join(_HERE, "libhp_b200.so")

HP_EINVAL = -1

c_p = ctypes.c_void_p
c_i64 = ctypes.c_int64
HP_ESPACE = -3  # hashpoint_b200.h
c_i32 = ctypes.c_int32
c_f64 = ctypes.c_double
c_size = ctypes.c_size_t


class Camera(ctypes.Structure):
    _fields_ = [("origin", c_f64 * 3), ("right", c_f64 * 3), ("up", c_f64 * 3),
                ("forward", c_f64 * 3), ("focal_length", c_f64), ("pixel_width", c_f64),
                ("pixel_height", c_f64), ("width", c_i64), ("height", c_i64)]


class Layout(ctypes.Structure):
    _fields_ = [("row_ptr", c_p), ("rel_x", c_p), ("rel_y", c_p), ("rel_z", c_p),
                ("point_id", c_p), ("relf", c_p), ("rel4", c_p)]


class SamplerParams(ctypes.Structure):
    _fields_ = [("k_neighbors", c_i32), ("eps_mode", c_i32), ("want_color", c_i32),
                ("exact_t_end", c_i32), ("beta2", c_f64), ("gamma", c_f64), ("eps", c_f64),
                ("tau_min", c_f64), ("emit_knn", c_i32), ("reserved", c_i32)]


class SampleFields(ctypes.Structure):
    _fields_ = [("r_id", c_p), ("r_t", c_p), ("r_dist", c_p), ("r_udf", c_p), ("r_alpha", c_p), ("r_w", c_p),
                ("r_color", c_p), ("r_knn_id", c_p), ("r_knn_w", c_p)]


class SamplePrefix(ctypes.Structure):
    _fields_ = [("start", c_p), ("length", c_p), ("ids", c_p), ("t", c_p), ("dist", c_p),
                ("cut_t", c_p), ("cut_d", c_p), ("u", c_p)]


_SIGNATURES = {
    "hp_last_error": (ctypes.c_char_p, []),
    "hp_version": (ctypes.c_int, []),
    "hp_launch_count": (c_i64, []),
    "hp_build_workspace_bytes": (ctypes.c_int, [c_i64, c_i64, c_i64, ctypes.POINTER(c_size)]),
    "hp_build_layout_workspace_bytes": (ctypes.c_int, [c_i64, c_i64, c_i64, ctypes.POINTER(c_size)]),
    "hp_build_layout": (ctypes.c_int, [c_p, c_i64, ctypes.POINTER(Camera), c_i64, c_i64, c_i64, Layout, c_p, c_p,
                                       c_size, c_p]),
    "hp_build": (ctypes.c_int, [c_p, c_i64, ctypes.POINTER(Camera), c_i64, c_p, c_p, c_p, c_p, c_p,
                                c_p, Layout, c_p, c_p, c_size, c_p]),
    "hp_scatter_by_bucket_workspace_bytes": (ctypes.c_int, [c_i64, c_i64, c_i64, ctypes.POINTER(c_size)]),
    "hp_scatter_by_bucket": (ctypes.c_int, [c_p, c_p, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_size, c_p]),
    "hp_layout_workspace_bytes": (ctypes.c_int, [c_i64, c_i64, c_i64, ctypes.POINTER(c_size)]),
    "hp_layout_from_table": (ctypes.c_int, [c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_i64, c_i64,
                                            ctypes.POINTER(c_f64), Layout, c_p, c_size, c_p]),
    "hp_radius_slopes_host": (ctypes.c_int, [ctypes.POINTER(Camera), c_p, c_i64, c_i64, c_f64, ctypes.c_int,
                                             c_p, ctypes.c_int]),
    "hp_radius_slopes": (ctypes.c_int, [ctypes.POINTER(Camera), c_i64, c_p, c_i64, c_i64, c_f64, ctypes.c_int,
                                        c_p, c_p]),
    "hp_host_upload": (ctypes.c_int, [c_p, c_p, c_size, c_p, c_size, ctypes.c_int, c_p]),
    "hp_splice_samples": (ctypes.c_int, [c_i64, c_p, c_p, c_p, c_p, ctypes.c_int32, ctypes.POINTER(SampleFields),
                                         ctypes.POINTER(SampleFields), ctypes.POINTER(SampleFields), c_p]),
    "hp_query_workspace_bytes": (ctypes.c_int, [c_i64, c_i64, c_i64, ctypes.POINTER(c_size)]),
    "hp_query_count": (ctypes.c_int, [Layout, ctypes.POINTER(Camera), c_i64, c_i64, c_i64, c_p, c_i64,
                                      c_p, c_p, c_p, c_p, c_i64, c_p, c_p, c_p, c_i64,
                                      c_p, c_size, c_p]),
    "hp_head_workspace_bytes": (ctypes.c_int, [c_i64, c_i64, ctypes.POINTER(c_size)]),
    "hp_head_count": (ctypes.c_int, [Layout, ctypes.POINTER(Camera), c_i64, c_i64, c_i64, c_p, c_i64,
                                     c_p, c_p, c_p, c_p, c_i64, c_p, c_p, c_p, c_p, c_i64,
                                     c_p, c_size, c_p]),
    "hp_head_sort": (ctypes.c_int, [Layout, c_p, c_p, c_i64, c_p, c_p, c_i64, c_p, ctypes.c_int32, ctypes.c_int32,
                                    c_p, c_p, c_p, c_p, c_p, c_p, c_p, ctypes.POINTER(SamplerParams), c_p, c_i64, c_p,
                                    c_size, c_p]),
    "hp_ray_grid": (ctypes.c_int, [ctypes.POINTER(Camera), c_i64, c_i64, c_p, c_p, ctypes.c_double,
                                   ctypes.c_double, c_p, c_p, c_p]),
    "hp_render": (ctypes.c_int, [ctypes.c_int, c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_i64, c_p,
                                 ctypes.c_int32, c_p, c_i64, c_i64, c_p, c_p, c_p, c_p]),
    "hp_query_bounds": (ctypes.c_int, [Layout, ctypes.POINTER(Camera), c_i64, c_i64, c_i64, c_p, c_i64,
                                       c_p, c_p, c_p, c_p, c_i64, c_p, c_p, c_size, c_p]),
    "hp_query_fill": (ctypes.c_int, [c_p, c_i64, c_i64, c_p, c_p, c_p, c_p, c_p, c_i64, c_p, c_size, c_p]),
    "hp_sample_workspace_bytes": (ctypes.c_int, [c_i64, c_i64, c_i64,
                                                 ctypes.POINTER(SamplerParams),
                                                 ctypes.POINTER(c_size)]),
    "hp_sample_run": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_p, c_i64, c_i64, c_p, c_p,
                                     ctypes.POINTER(SamplerParams), c_p, c_i64, c_p, c_p,
                                     c_p, c_size, c_p]),
    "hp_sample_emit": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_p, c_i64, c_i64, c_p,
                                      ctypes.POINTER(SamplerParams), c_p, c_i64, c_p, c_i64,
                                      c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_size, c_p]),
    "hp_sample_run_prefix": (ctypes.c_int, [c_p, c_i64, ctypes.POINTER(SamplePrefix), c_i64, c_p, c_p,
                                            ctypes.POINTER(SamplerParams), c_p, c_i64, c_p, c_p, c_p, c_p,
                                            c_size, c_p]),
    "hp_sample_emit_prefix": (ctypes.c_int, [c_p, c_i64, ctypes.POINTER(SamplePrefix), c_i64, c_p,
                                             ctypes.POINTER(SamplerParams), c_p, c_i64, c_p, c_i64,
                                             c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_size, c_p]),
    "hp_pointnerf_aggregate": (ctypes.c_int, [c_p, c_p, c_i64, ctypes.c_int32, c_p, c_p, c_p,
                                              ctypes.POINTER(c_f64), c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
    "hp_pointnerf_head": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_p, c_p, c_p, c_p]),
    "hp_csr_stats": (ctypes.c_int, [c_p, c_i64, c_p, c_p]),
    "hp_primary_surface": (ctypes.c_int, [c_p, c_i64, c_p, c_p, c_p, c_p, c_p]),
    "hp_sample_debug_counters": (ctypes.c_int, [c_p, ctypes.c_int]),
    "hp_check_failures": (ctypes.c_int, [c_p, ctypes.c_int, ctypes.c_int]),
    "hp_timing_enable": (ctypes.c_int, [ctypes.c_int]),
    "hp_timing_collect": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, c_p, c_p, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_int)]),
}

EXPORTS = tuple(_SIGNATURES)

_lib = None


def load(require_device: bool = False):
    """Load the shared library (no GPU needed just to load it)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    if require_device:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2404_14044_b200 needs a CUDA device (B200, sm_100a); "
                               "there is no CPU fallback")
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (_lib.hp_last_error() or b"").decode()
    if rc == HP_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def launch_count() -> int:
    return int(load().hp_launch_count())


def timing_enable(on: bool) -> None:
    check(load().hp_timing_enable(1 if on else 0))


def timing_collect() -> dict:
    """{kernel name: (summed ms, launches)} since the last collect (syncs)."""
    import numpy as np
    L = load()
    names = ctypes.create_string_buffer(4096)
    ms = np.zeros(64)
    cnt = np.zeros(64, np.int64)
    n = ctypes.c_int(0)
    check(L.hp_timing_collect(names, 4096, ms.ctypes.data_as(c_p), cnt.ctypes.data_as(c_p), 64,
                              ctypes.byref(n)))
    keys = names.value.decode().split("\n")[: n.value]
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(keys)}


def check_failures(reset: bool = True) -> list:
    """Checked build: source lines of failed device-side checks (empty
    otherwise)."""
    import numpy as np
    out = np.zeros(16, np.int64)
    n = load().hp_check_failures(out.ctypes.data_as(c_p), 16, 1 if reset else 0)
    if n < 0:
        check(n)
    return [int(x) for x in out[: min(n, 16)]]
