"""The reference's operator layer (hashpoint/_kernels.py) on the device, with
its exact signatures: C-contiguous numpy arrays in, freshly allocated numpy
arrays out (``scatter_by_bucket`` mutates ``cursor`` and ``out_ids`` in
place, like the reference).  This is the plugin boundary a maintainer swaps
in for the numba kernels: every call goes through
libhp_b200.so (sm_100a); there is no CPU fallback.

  scatter_by_bucket   _kernels.py:76-83    -> hp_scatter_by_bucket
  hash_query_batch    _kernels.py:86-157   -> hp_layout_from_table + hp_query_count / hp_query_fill
  sample_batch        _kernels.py:552-700  -> hp_sample_run / hp_sample_emit
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib, device

__all__ = ["scatter_by_bucket", "hash_query_batch", "sample_batch"]


def _dev():
    _lib.load(require_device=True)
    return torch.device("cuda", torch.cuda.current_device())


def _up(a, dtype, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(dev)


def scatter_by_bucket(buckets, orig_ids, cursor, out_ids):
    """Counting-sort placement pass: stable within a bucket by input order
    (reference _kernels.py:76-83).  ``cursor`` (int64 [P]) and ``out_ids``
    (int64) are updated in place."""
    if not (isinstance(cursor, np.ndarray) and isinstance(out_ids, np.ndarray)
            and cursor.dtype == np.int64 and out_ids.dtype == np.int64
            and cursor.flags.c_contiguous and out_ids.flags.c_contiguous):
        raise ValueError("cursor and out_ids must be C-contiguous int64 numpy arrays (updated in place)")
    b = np.ascontiguousarray(buckets, dtype=np.int64)
    n = b.shape[0]
    if n == 0:
        return
    P, n_out = cursor.shape[0], out_ids.shape[0]
    if b.min() < 0 or b.max() >= P:
        raise ValueError("bucket index out of range")
    cnt = np.bincount(b, minlength=P)
    if np.any(cursor[cnt > 0] < 0) or np.any(cursor + cnt > n_out):
        raise ValueError("cursor ranges exceed out_ids")
    dev = _dev()
    lib = _lib.load()
    nb = _lib.c_size(0)
    _lib.check(lib.hp_scatter_by_bucket_workspace_bytes(n, P, n_out, ctypes.byref(nb)))
    ws = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=dev)
    cur = _up(cursor, np.int64, dev)
    out = _up(out_ids, np.int64, dev)
    bd, od = _up(b, np.int64, dev), _up(orig_ids, np.int64, dev)  # alive until the kernels have run
    _lib.check(lib.hp_scatter_by_bucket(device._ptr(bd), device._ptr(od), n, device._ptr(cur), P, device._ptr(out),
                                        n_out, device._ptr(ws), nb.value, device._stream()))
    cursor[...] = cur.cpu().numpy()
    out_ids[...] = out.cpu().numpy()


class _TableCamera:
    """Just what the device index needs from a camera when it is built from
    a table: the unpadded size and the origin (no footprint: every pixel of
    the s x s window is probed, as the reference kernel)."""

    def __init__(self, padded_w, padded_h, pad, origin):
        self.width, self.height = padded_w - 2 * pad, padded_h - 2 * pad
        self.origin = np.asarray(origin, np.float64)


def hash_query_batch(table_start, table_count, slot_x, slot_y, slot_z, slot_ids, padded_w, pad, px_u, px_v, dirs,
                     origin, t_near, t_far, slopes):
    """Probe the s*s kernel around each ray's pixel and cone-test its points
    (reference _kernels.py:86-157).  Returns ``(offsets, ids, t_proj,
    dist_perp, probes, scanned)``, bit-identical to the reference."""
    dev = _dev()
    ts = _up(table_start, np.int64, dev)
    P, wp, pad = ts.shape[0], int(padded_w), int(pad)
    if wp <= 0 or P % wp:
        raise ValueError("table size is not a multiple of padded_w")
    cam = _TableCamera(wp, P // wp, pad, origin)
    idx = device.build_from_table(ts, _up(table_count, np.int64, dev), _up(slot_x, np.float64, dev),
                                  _up(slot_y, np.float64, dev), _up(slot_z, np.float64, dev),
                                  _up(slot_ids, np.int64, dev), cam, pad)
    px = np.stack([np.asarray(px_u, np.int64), np.asarray(px_v, np.int64)], axis=1)
    out = device.query(idx, _up(px, np.int64, dev), _up(np.asarray(dirs).reshape(-1, 3), np.float64, dev),
                       _up(t_near, np.float64, dev), _up(t_far, np.float64, dev), _up(slopes, np.float64, dev),
                       footprint=False)
    return tuple(x.cpu().numpy() for x in out)


def sample_batch(offsets, ids, ts, ds, slopes, k_neighbors, beta2, gamma, eps_mode, eps, tau_min, colors,
                 want_color):
    """Full per-ray sampling pipeline over CSR query results (reference
    _kernels.py:552-700): ``(r_off, r_id, r_t, r_dist, r_udf, r_alpha, r_w,
    r_color, t_end)``; r_color is (R, 3) when ``want_color`` else ``colors``'
    (0, 3) shape, as the reference."""
    dev = _dev()
    p = _lib.SamplerParams()
    p.k_neighbors, p.eps_mode = int(k_neighbors), 1 if eps_mode else 0
    p.beta2, p.gamma, p.eps, p.tau_min = float(beta2), float(gamma), float(eps), float(tau_min)
    col = _up(np.asarray(colors).reshape(-1, 3), np.float64, dev) if want_color else None
    out = device.sample(_up(offsets, np.int64, dev), _up(ids, np.int64, dev), _up(ts, np.float64, dev),
                        _up(ds, np.float64, dev), _up(slopes, np.float64, dev), p, col)
    res = [x.cpu().numpy() for x in out]
    if not want_color:
        res[7] = np.empty((0, 3), np.float64)
    return tuple(res)
