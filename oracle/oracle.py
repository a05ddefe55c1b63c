"""ctypes wrapper of the C oracle (``oracle/libhp_oracle.so``).

TEST INFRASTRUCTURE ONLY: the parity checker for tests/, smoke() and the CPU
baseline legs of bench.py.  The product package never imports this module.

Functions mirror the reference operator layer:
  build            hash_index.build            (hash_index.py:151-190)
  query            _kernels.hash_query_batch   (_kernels.py:86-157)
  sample           _kernels.sample_batch       (_kernels.py:552-700)
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libhp_oracle.so")
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_INT = ctypes.c_int


def build_library() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build_library()
        L = ctypes.CDLL(_LIB_PATH)
        L.hpo_build.restype = _I64
        L.hpo_build.argtypes = [_P, _I64, _P, _I64, _P, _P, _P, _P, _P, _P]
        L.hpo_rasterize.restype = None
        L.hpo_rasterize.argtypes = [_P, _I64, _P, _I64, _P]
        L.hpo_morton.restype = _I64
        L.hpo_morton.argtypes = [_I64, _I64]
        L.hpo_query_run.restype = _P
        L.hpo_query_run.argtypes = [_P, _P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P,
                                    _P, _P, _I64, _INT, ctypes.POINTER(_I64)]
        L.hpo_query_take.restype = None
        L.hpo_query_take.argtypes = [_P] * 7
        L.hpo_sample_run.restype = _P
        L.hpo_sample_run.argtypes = [_P, _I64, _P, _P, _P, _P, _INT, _D, _D, _INT, _D, _D,
                                     _P, _INT, _INT, ctypes.POINTER(_I64)]
        L.hpo_sample_take.restype = None
        L.hpo_sample_take.argtypes = [_P] * 10
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def camera_block(camera) -> np.ndarray:
    """Flat camera record: origin, right, up, forward, f, pw, ph, W, H."""
    return np.concatenate([
        np.asarray(camera.origin, np.float64), np.asarray(camera.orientation, np.float64).ravel(),
        [camera.focal_length, camera.pixel_width, camera.pixel_height,
         float(camera.width), float(camera.height)]]).astype(np.float64)


def rasterize(positions, camera, pad):
    xyz = _c(positions, np.float64).reshape(-1, 3)
    lin = np.empty(xyz.shape[0], np.int64)
    cam = camera_block(camera)
    lib().hpo_rasterize(_ptr(xyz), xyz.shape[0], _ptr(cam), int(pad), _ptr(lin))
    return lin


def build(positions, camera, pad):
    """Returns dict(table_start, table_count, reordered_ids, slot_x, slot_y, slot_z)."""
    xyz = _c(positions, np.float64).reshape(-1, 3)
    n = xyz.shape[0]
    wp, hp = camera.width + 2 * pad, camera.height + 2 * pad
    P = wp * hp
    ts = np.empty(P, np.int64)
    tc = np.empty(P, np.int64)
    ids = np.empty(max(n, 1), np.int64)
    sx, sy, sz = (np.empty(max(n, 1)) for _ in range(3))
    cam = camera_block(camera)
    n_in = lib().hpo_build(_ptr(xyz), n, _ptr(cam), int(pad), _ptr(ts), _ptr(tc), _ptr(ids),
                           _ptr(sx), _ptr(sy), _ptr(sz))
    return dict(table_start=ts, table_count=tc, reordered_ids=ids[:n_in].copy(),
                slot_x=sx[:n_in].copy(), slot_y=sy[:n_in].copy(), slot_z=sz[:n_in].copy())


def query(table_start, table_count, slot_x, slot_y, slot_z, slot_ids, padded_w, pad,
          px_u, px_v, dirs, origin, t_near, t_far, slopes, threads=1):
    """Same argument list and 6-tuple result as ``_kernels.hash_query_batch``."""
    args = [_c(table_start, np.int64), _c(table_count, np.int64), _c(slot_x, np.float64),
            _c(slot_y, np.float64), _c(slot_z, np.float64), _c(slot_ids, np.int64)]
    pu, pv = _c(px_u, np.int64), _c(px_v, np.int64)
    dirs = _c(dirs, np.float64).reshape(-1, 3)
    o = _c(origin, np.float64)
    tn, tf, sl = _c(t_near, np.float64), _c(t_far, np.float64), _c(slopes, np.float64)
    m = pu.shape[0]
    total = _I64(0)
    h = lib().hpo_query_run(*[_ptr(a) for a in args], int(padded_w), int(pad), _ptr(pu), _ptr(pv),
                            _ptr(dirs), _ptr(o), _ptr(tn), _ptr(tf), _ptr(sl), m, int(threads),
                            ctypes.byref(total))
    Q = total.value
    off = np.empty(m + 1, np.int64)
    ids = np.empty(Q, np.int64)
    t = np.empty(Q)
    d = np.empty(Q)
    probes = np.empty(m, np.int64)
    scanned = np.empty(m, np.int64)
    lib().hpo_query_take(h, _ptr(off), _ptr(ids), _ptr(t), _ptr(d), _ptr(probes), _ptr(scanned))
    return off, ids, t, d, probes, scanned


def sample(offsets, ids, ts, ds, slopes, k_neighbors, beta2, gamma, eps_mode, eps, tau_min,
           colors=None, threads=1):
    """Same argument meaning and 9-tuple result as ``_kernels.sample_batch``."""
    off = _c(offsets, np.int64)
    ids = _c(ids, np.int64)
    ts = _c(ts, np.float64)
    ds = _c(ds, np.float64)
    sl = _c(slopes, np.float64)
    want = colors is not None
    col = _c(colors, np.float64).reshape(-1, 3) if want else None
    m = off.shape[0] - 1
    total = _I64(0)
    h = lib().hpo_sample_run(_ptr(off), m, _ptr(ids), _ptr(ts), _ptr(ds), _ptr(sl),
                             int(k_neighbors), float(beta2), float(gamma), int(bool(eps_mode)),
                             float(eps), float(tau_min), _ptr(col), int(want), int(threads),
                             ctypes.byref(total))
    R = total.value
    r_off = np.empty(m + 1, np.int64)
    out = [np.empty(R, np.int64)] + [np.empty(R) for _ in range(5)]
    r_color = np.empty((R, 3)) if want else np.zeros((0, 3))
    t_end = np.empty(m)
    lib().hpo_sample_take(h, _ptr(r_off), *[_ptr(a) for a in out],
                          _ptr(r_color) if want else None, _ptr(t_end))
    return (r_off, *out, r_color, t_end)
