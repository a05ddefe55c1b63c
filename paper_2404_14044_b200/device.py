"""Device-resident pipeline: torch CUDA tensors in, torch CUDA tensors out.

These are the functions the drop-in wrappers (hash_index.py, sampler.py) and
the benchmark call.  Each one enqueues the sm_100a kernels of libhp_b200.so on
torch's current CUDA stream through the C ABI; torch only provides device
memory, streams and the host<->device copies.  Host synchronisation happens
only where a size must be known to allocate an output (N_in after the build,
Q after the query count pass, R after the sampler), as in the two-phase C ABI.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib
from ._lib import c_size

__all__ = ["DeviceIndex", "build", "build_from_table", "query", "query_bounds", "query_prefix", "query_frame", "sample", "sample_prefix", "merge_flagged", "ray_grid",
           "primary_surface", "MatchBudgetExceeded", "SAMPLE_EXACT_PER_RAY"]

# match-scratch capacity of the last query per device (slots), reused so a
# steady stream of frames sizes its workspace once
_QUERY_CAP: dict = {}
SAMPLE_EXACT_PER_RAY = 16  # initial exact-candidate scratch per ray (grown on demand)

# Optional per-kernel timer (pipeline.StageTimer); set by the benchmark.
TIMER = None


def _mark(name):
    if TIMER is not None:
        TIMER.mark(name)


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _host_read(*vals) -> list:
    """Host values of scalar device tensors (one synchronisation): copied into
    pinned memory and waited for with an event -- a pageable read holds the
    driver while it waits, stalling other threads' uploads (the host-buffer
    entry points stage the next chunk's rays on a thread meanwhile)."""
    t = torch.stack([v.reshape(()).to(torch.int64) for v in vals])
    h = torch.empty(t.shape, dtype=torch.int64, pin_memory=True)
    h.copy_(t, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    ev.synchronize()
    return [int(x) for x in h.tolist()]


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def camera_struct(camera) -> _lib.Camera:
    c = _lib.Camera()
    o = np.asarray(camera.origin, np.float64)
    rot = np.asarray(camera.orientation, np.float64)
    for k in range(3):
        c.origin[k] = float(o[k])
        c.right[k] = float(rot[0, k])
        c.up[k] = float(rot[1, k])
        c.forward[k] = float(rot[2, k])
    c.focal_length = float(camera.focal_length)
    c.pixel_width = float(camera.pixel_width)
    c.pixel_height = float(camera.pixel_height)
    c.width = int(camera.width)
    c.height = int(camera.height)
    return c


class DeviceIndex:
    """Hash index in HBM: the reference's HashIndex arrays plus the row-major
    query layout (origin-relative fp64 coordinates, int32 ids, row pointers,
    fp32 filter copy).  Arrays are allocated with capacity n; N_in is read
    from the device only when first needed (no synchronisation in build)."""

    def __init__(self, camera, pad, padded_width, padded_height, n_in_dev, table_start, table_count,
                 reordered_ids, slot_x, slot_y, slot_z, row_ptr, rel_x, rel_y, rel_z, point_id, relf,
                 rel4, n_in=None):
        self.camera = camera
        self.pad = pad
        self.padded_width = padded_width
        self.padded_height = padded_height
        self._n_in_dev = n_in_dev
        self._n_in = n_in
        self.table_start, self.table_count = table_start, table_count
        self._rid, self._sx, self._sy, self._sz = reordered_ids, slot_x, slot_y, slot_z
        self.row_ptr, self.rel_x, self.rel_y, self.rel_z = row_ptr, rel_x, rel_y, rel_z
        self.point_id, self.relf, self.rel4 = point_id, relf, rel4

    @property
    def n_in(self) -> int:
        if self._n_in is None:
            self._n_in = int(self._n_in_dev.item())
        return self._n_in

    reordered_ids = property(lambda self: self._rid[: self.n_in])
    slot_x = property(lambda self: self._sx[: self.n_in])
    slot_y = property(lambda self: self._sy[: self.n_in])
    slot_z = property(lambda self: self._sz[: self.n_in])

    @property
    def device(self) -> torch.device:
        return self.row_ptr.device

    def layout(self) -> _lib.Layout:
        return _lib.Layout(_ptr(self.row_ptr), _ptr(self.rel_x), _ptr(self.rel_y),
                           _ptr(self.rel_z), _ptr(self.point_id), _ptr(self.relf), _ptr(self.rel4))


def build(positions: torch.Tensor, camera, pad: int) -> DeviceIndex:
    """hash_index.build on the device (reference hash_index.py:151-190)."""
    lib = _lib.load(require_device=True)
    pad = int(pad)
    wp, hp = int(camera.width) + 2 * pad, int(camera.height) + 2 * pad
    if max(wp, hp) > 0xFFFF:
        raise ValueError("padded image exceeds 16-bit pixel coordinates")
    dev = positions.device
    xyz = positions.contiguous().view(-1, 3)
    n = xyz.shape[0]
    P = wp * hp
    nb = c_size(0)
    _lib.check(lib.hp_build_workspace_bytes(n, wp, hp, ctypes.byref(nb)))
    ws = _workspace(nb.value, dev)
    i64 = dict(dtype=torch.int64, device=dev)
    f64 = dict(dtype=torch.float64, device=dev)
    ts, tc = torch.empty(P, **i64), torch.empty(P, **i64)
    cap = max(n, 1)
    rid = torch.empty(cap, **i64)
    sx, sy, sz = (torch.empty(cap, **f64) for _ in range(3))
    row_ptr = torch.empty(P + 1, dtype=torch.int32, device=dev)
    rx, ry, rz = (torch.empty(cap, **f64) for _ in range(3))
    pid = torch.empty(cap, dtype=torch.int32, device=dev)
    rf = torch.empty((cap, 4), dtype=torch.float32, device=dev)
    r4 = torch.empty((cap, 4), **f64)
    n_in_d = torch.zeros(1, **i64)
    _mark("build.setup")
    L = _lib.Layout(_ptr(row_ptr), _ptr(rx), _ptr(ry), _ptr(rz), _ptr(pid), _ptr(rf), _ptr(r4))
    cam = camera_struct(camera)
    _lib.check(lib.hp_build(_ptr(xyz), n, ctypes.byref(cam), pad, _ptr(ts), _ptr(tc), _ptr(rid),
                            _ptr(sx), _ptr(sy), _ptr(sz), L, _ptr(n_in_d), _ptr(ws), nb.value,
                            _stream()))
    _mark("build.kernels")
    return DeviceIndex(camera, pad, wp, hp, n_in_d, ts, tc, rid, sx, sy, sz, row_ptr, rx, ry, rz,
                       pid, rf, r4, n_in=0 if n == 0 else None)


def build_layout(positions: torch.Tensor, camera, pad: int, rows: tuple | None = None) -> DeviceIndex:
    """The query layout alone (hp_build_layout): what a frame that only
    queries needs, without the reference's HashIndex arrays (table_start ...
    are None).  ``rows``: (a, b) image rows of the frame's rays -- only points
    in the padded rows those rays reach, [a, b + 2 pad), are placed.  Inside a
    pixel the order is arbitrary (the query ranks by (t, id))."""
    lib = _lib.load(require_device=True)
    pad = int(pad)
    wp, hp = int(camera.width) + 2 * pad, int(camera.height) + 2 * pad
    if max(wp, hp) > 0xFFFF:
        raise ValueError("padded image exceeds 16-bit pixel coordinates")
    dev = positions.device
    xyz = positions.contiguous().view(-1, 3)
    n = xyz.shape[0]
    P = wp * hp
    nb = c_size(0)
    _lib.check(lib.hp_build_layout_workspace_bytes(n, wp, hp, ctypes.byref(nb)))
    ws = _workspace(nb.value, dev)
    cap = max(n, 1)
    f64 = dict(dtype=torch.float64, device=dev)
    row_ptr = torch.empty(P + 1, dtype=torch.int32, device=dev)
    rx, ry, rz = (torch.empty(cap, **f64) for _ in range(3))
    pid = torch.empty(cap, dtype=torch.int32, device=dev)
    rf = torch.empty((cap, 4), dtype=torch.float32, device=dev)
    r4 = torch.empty((cap, 4), **f64)
    n_in_d = torch.zeros(1, dtype=torch.int64, device=dev)
    r0, r1 = (0, 0) if rows is None else (int(rows[0]), int(rows[1]) + 2 * pad)
    _mark("build.setup")
    L = _lib.Layout(_ptr(row_ptr), _ptr(rx), _ptr(ry), _ptr(rz), _ptr(pid), _ptr(rf), _ptr(r4))
    cam = camera_struct(camera)
    _lib.check(lib.hp_build_layout(_ptr(xyz), n, ctypes.byref(cam), pad, r0, r1, L, _ptr(n_in_d), _ptr(ws),
                                   nb.value, _stream()))
    _mark("build.kernels")
    return DeviceIndex(camera, pad, wp, hp, n_in_d, None, None, None, None, None, None, row_ptr, rx, ry, rz,
                       pid, rf, r4, n_in=0 if n == 0 else None)


def build_from_table(table_start, table_count, slot_x, slot_y, slot_z, reordered_ids, camera,
                     pad: int) -> DeviceIndex:
    """Device index from HashIndex arrays built elsewhere (e.g. by the reference)."""
    lib = _lib.load(require_device=True)
    dev = table_start.device
    pad = int(pad)
    wp, hp = int(camera.width) + 2 * pad, int(camera.height) + 2 * pad
    P = wp * hp
    n_in = int(reordered_ids.numel())
    cap = max(n_in, 1)
    row_ptr = torch.empty(P + 1, dtype=torch.int32, device=dev)
    rx, ry, rz = (torch.empty(cap, dtype=torch.float64, device=dev) for _ in range(3))
    pid = torch.empty(cap, dtype=torch.int32, device=dev)
    rf = torch.empty((cap, 4), dtype=torch.float32, device=dev)
    r4 = torch.empty((cap, 4), dtype=torch.float64, device=dev)
    nb = c_size(0)
    _lib.check(lib.hp_layout_workspace_bytes(n_in, wp, hp, ctypes.byref(nb)))
    ws = _workspace(nb.value, dev)
    origin = (ctypes.c_double * 3)(*[float(v) for v in np.asarray(camera.origin)])
    L = _lib.Layout(_ptr(row_ptr), _ptr(rx), _ptr(ry), _ptr(rz), _ptr(pid), _ptr(rf), _ptr(r4))
    _lib.check(lib.hp_layout_from_table(_ptr(table_start), _ptr(table_count), _ptr(slot_x),
                                        _ptr(slot_y), _ptr(slot_z), _ptr(reordered_ids), n_in, wp,
                                        hp, origin, L, _ptr(ws), nb.value, _stream()))
    return DeviceIndex(camera, pad, wp, hp, None, table_start, table_count, reordered_ids, slot_x,
                       slot_y, slot_z, row_ptr, rx, ry, rz, pid, rf, r4, n_in=n_in)


class MatchBudgetExceeded(RuntimeError):
    """The query's match scratch would exceed ``max_scratch`` slots."""

    def __init__(self, needed: int, budget: int):
        super().__init__(f"query needs {needed} match slots, budget {budget}")
        self.needed = needed
        self.budget = budget


def query_bounds(index: DeviceIndex, pixels: torch.Tensor, dirs: torch.Tensor, t_near: torch.Tensor,
                 t_far: torch.Tensor, slopes: torch.Tensor, footprint: bool = True) -> torch.Tensor:
    """Exclusive scan of the per-ray match upper bounds (hp_query_bounds),
    int64 [m+1]; used to split a frame into ray chunks that fit memory."""
    lib = _lib.load(require_device=True)
    dev = index.row_ptr.device
    m = int(pixels.shape[0])
    pixels, dirs = pixels.contiguous(), dirs.contiguous()
    nb = c_size(0)
    _lib.check(lib.hp_query_workspace_bytes(m, index.pad, 0, ctypes.byref(nb)))
    ws = _workspace(nb.value, dev)
    out = torch.empty(m + 1, dtype=torch.int64, device=dev)
    cam = ctypes.byref(camera_struct(index.camera)) if footprint else None
    _lib.check(lib.hp_query_bounds(index.layout(), cam, index.padded_width, index.padded_height, index.pad,
                                   _ptr(pixels), 2, _ptr(dirs), _ptr(t_near), _ptr(t_far), _ptr(slopes), m,
                                   _ptr(out), _ptr(ws), nb.value, _stream()))
    return out


def _count(index, pixels, dirs, t_near, t_far, slopes, footprint, max_scratch):
    """hp_query_count with the workspace sized (retrying once); returns
    (offsets, probes, scanned, total, workspace, workspace bytes, capacity)."""
    lib = _lib.load(require_device=True)
    dev = index.row_ptr.device
    m = int(pixels.shape[0])
    nb = c_size(0)
    offsets = torch.empty(m + 1, dtype=torch.int64, device=dev)
    probes = torch.empty(m, dtype=torch.int64, device=dev)
    scanned = torch.empty(m, dtype=torch.int64, device=dev)
    L = index.layout()
    cam = ctypes.byref(camera_struct(index.camera)) if footprint else None
    args = (L, cam, index.padded_width, index.padded_height, index.pad, _ptr(pixels), 2, _ptr(dirs),
            _ptr(t_near), _ptr(t_far), _ptr(slopes), m)
    # the frame size seen so far, but no more than a generous per-ray guess for
    # a much smaller query (e.g. the re-run of a frame's flagged rays)
    cap = min(_QUERY_CAP.get(dev, 0), 4096 * max(m, 1))
    if max_scratch is not None:
        cap = min(cap, int(max_scratch))
    _mark("query.setup")
    for _ in range(2):
        _lib.check(lib.hp_query_workspace_bytes(m, index.pad, cap, ctypes.byref(nb)))
        ws = _workspace(nb.value, dev)
        _lib.check(lib.hp_query_count(*args, _ptr(offsets), _ptr(probes), _ptr(scanned), cap, _ptr(ws),
                                      nb.value, _stream()))
        _mark("query.count")
        total = _host_read(offsets[m])[0]
        if total >= 0:
            break
        if _ == 1:
            raise RuntimeError(f"hp_query_count: scratch of {cap} slots still short ({-total} needed)")
        needed = -total  # scratch too small: nothing was written, grow it once (and remember)
        if max_scratch is not None and needed > max_scratch:
            raise MatchBudgetExceeded(needed, int(max_scratch))
        cap = int(needed * 1.0625) + 1024
        if max_scratch is not None:
            cap = min(cap, int(max_scratch))
        if cap > _QUERY_CAP.get(dev, 0):  # only grow: a small query (e.g. the re-run of a
            _QUERY_CAP[dev] = cap         # frame's flagged rays) must not shrink the frame's size
    return offsets, probes, scanned, total, ws, nb.value, cap


def query(index: DeviceIndex, pixels: torch.Tensor, dirs: torch.Tensor, t_near: torch.Tensor,
          t_far: torch.Tensor, slopes: torch.Tensor, footprint: bool = True, facts: bool = False,
          max_scratch: int | None = None):
    """_kernels.hash_query_batch on the device (reference _kernels.py:86-157).

    Returns (offsets, ids, t_proj, dist_perp, probes, scanned) as CUDA tensors
    (+ the per-ray sampler facts, int32 [m], with ``facts=True``; pass them to
    :func:`sample` together with this CSR and these slopes).  With
    ``max_scratch`` a frame needing more match slots raises
    :class:`MatchBudgetExceeded` before any CSR is written.
    """
    pixels, dirs = pixels.contiguous(), dirs.contiguous()
    return _fill(index, _count(index, pixels, dirs, t_near, t_far, slopes, footprint, max_scratch), slopes,
                 facts)


def _fill(index, counted, slopes, facts):
    """hp_query_fill after :func:`_count`: the (t, id)-sorted CSR."""
    lib = _lib.load(require_device=True)
    dev = index.row_ptr.device
    offsets, probes, scanned, total, ws, nb, cap = counted
    m = int(offsets.shape[0]) - 1
    ids = torch.empty(total, dtype=torch.int64, device=dev)
    t = torch.empty(total, dtype=torch.float64, device=dev)
    d = torch.empty(total, dtype=torch.float64, device=dev)
    _mark("query.sync")
    fa = torch.empty(m, dtype=torch.int32, device=dev) if facts else None
    _lib.check(lib.hp_query_fill(_ptr(offsets), m, total, _ptr(ids), _ptr(t), _ptr(d),
                                 _ptr(slopes) if facts else ctypes.c_void_p(0),
                                 _ptr(fa) if facts else ctypes.c_void_p(0), cap, _ptr(ws), nb, _stream()))
    _mark("query.fill")
    if facts:
        return offsets, ids, t, d, probes, scanned, fa
    return offsets, ids, t, d, probes, scanned


class QueryPrefix:
    """Result of :func:`query_prefix`: the full match counts (``offsets``)
    and, per ray, the (t, id)-sorted head of its matches (``start``,
    ``length``; ``t``, ``ids`` int32, ``dist``), lower bounds of the t / dist
    of the matches left out (``cut_t``, ``cut_d``), and the sampler's facts
    over the head.  Keeps the query workspace alive."""

    def __init__(self, offsets, probes, scanned, start, length, t, ids, dist, cut_t, cut_d, facts, ws, u=None):
        self.offsets, self.probes, self.scanned = offsets, probes, scanned
        self.start, self.length, self.t, self.ids, self.dist = start, length, t, ids, dist
        self.cut_t, self.cut_d, self.facts = cut_t, cut_d, facts
        self.u = u  # precomputed bound factors (float32, next to t) or None
        self._ws = ws

    def struct(self) -> _lib.SamplePrefix:
        sp = _lib.SamplePrefix()
        sp.start, sp.length, sp.ids = self.start.data_ptr(), self.length.data_ptr(), self.ids.data_ptr()
        sp.t, sp.dist = self.t.data_ptr(), self.dist.data_ptr()
        sp.cut_t, sp.cut_d = self.cut_t.data_ptr(), self.cut_d.data_ptr()
        sp.u = self.u.data_ptr() if self.u is not None else None
        return sp


PREFIX_WANT = int(os.environ.get("HP_PREFIX_WANT", "400"))  # head length the sampler usually needs
HEAD_CAP = 1024  # longest head (hp_head.cu kHeadCap)
HEAD_LONG = 4096  # the long-head mode of a re-sort (hp_head.cu kHeadLong)
# HP_HEAD_FACTORS=1: heads carry the sampler's bound factors (measured: the sort pays more than the plan saves)
HEAD_FACTORS = os.environ.get("HP_HEAD_FACTORS", "0") == "1"
# rays of at most this many matches are sorted whole; longer ones are cut near PREFIX_WANT
HEAD_WHOLE = int(os.environ.get("HP_HEAD_WHOLE", "512"))


class CountShort(Exception):
    """A deferred head count (no host read between hp_head_count and the
    sampler) ran short of scratch: re-run the frame's query synchronously."""


# Frames enqueue hp_head_count -> hp_head_sort -> the sampler with no host
# read in between once a scratch size is known for the device (the head
# arrays then sized by that capacity; Q and a short count are checked at the
# sampler's read).  False: read Q after the count, as a first frame does.
DEFER_COUNT = os.environ.get("HP_DEFER_COUNT", "1") != "0"
_DEFER_OK: dict = {}  # per device: False after a deferred count ran short / a frame needed chunks


def _count_head(index, pixels, dirs, t_near, t_far, slopes, footprint, max_scratch, defer=False, frame=False):
    """hp_head_count with the workspace sized (retrying once); returns
    (offsets, head_off, probes, scanned, Q, head capacity, workspace, bytes,
    capacity) -- Q and the head capacity read in one synchronisation.
    ``defer``: no read when a scratch size is known (Q None, head capacity =
    the scratch capacity; the caller checks offsets[m] later).  ``frame``: a
    whole frame's count (its outcome decides whether later frames defer)."""
    lib = _lib.load(require_device=True)
    dev = index.row_ptr.device
    m = int(pixels.shape[0])
    nb = c_size(0)
    offsets = torch.empty(m + 1, dtype=torch.int64, device=dev)
    head_off = torch.empty(m + 1, dtype=torch.int64, device=dev)
    probes = torch.empty(m, dtype=torch.int64, device=dev)
    scanned = torch.empty(m, dtype=torch.int64, device=dev)
    cam = ctypes.byref(camera_struct(index.camera)) if footprint else None
    args = (index.layout(), cam, index.padded_width, index.padded_height, index.pad, _ptr(pixels), 2,
            _ptr(dirs), _ptr(t_near), _ptr(t_far), _ptr(slopes), m)
    cap = min(_QUERY_CAP.get(dev, 0), 4096 * max(m, 1))
    if max_scratch is not None:
        cap = min(cap, int(max_scratch))
    _mark("query.setup")
    if defer and cap > 0 and _DEFER_OK.get(dev, True):
        _lib.check(lib.hp_head_workspace_bytes(m, cap, ctypes.byref(nb)))
        ws = _workspace(nb.value, dev)
        _lib.check(lib.hp_head_count(*args, _ptr(offsets), _ptr(head_off), _ptr(probes), _ptr(scanned), cap,
                                     _ptr(ws), nb.value, _stream()))
        _mark("query.count")
        # head arrays: sum_r min(q_r, 1024) <= min(Q, 1024 m)
        return offsets, head_off, probes, scanned, None, min(cap, HEAD_CAP * max(m, 1)), ws, nb.value, cap
    # read first: the exact scratch need from the (cheap) bound pass -- a
    # count over a short capacity still streams every group placed below it
    need = _host_read(query_bounds(index, pixels, dirs, t_near, t_far, slopes, footprint)[m])[0]
    if max_scratch is not None and need > max_scratch:
        if frame:
            _DEFER_OK[dev] = False  # frames of this size run in chunks
        raise MatchBudgetExceeded(need, int(max_scratch))
    cap = int(need * 1.0625) + 1024  # headroom for the next (deferred) frame
    if max_scratch is not None:
        cap = max(min(cap, int(max_scratch)), need)
    if cap > _QUERY_CAP.get(dev, 0):
        _QUERY_CAP[dev] = cap
    for _ in range(2):
        _lib.check(lib.hp_head_workspace_bytes(m, cap, ctypes.byref(nb)))
        ws = _workspace(nb.value, dev)
        _lib.check(lib.hp_head_count(*args, _ptr(offsets), _ptr(head_off), _ptr(probes), _ptr(scanned), cap,
                                     _ptr(ws), nb.value, _stream()))
        _mark("query.count")
        total, hcap = _host_read(offsets[m], head_off[m])  # one synchronisation
        if total >= 0:
            if _ == 0 and frame:
                _DEFER_OK[dev] = True  # the remembered size fits: later frames may defer the read
            break
        if _ == 1:
            raise RuntimeError(f"hp_head_count: scratch of {cap} slots still short ({-total} needed)")
        needed = -total
        if max_scratch is not None and needed > max_scratch:
            if frame:
                _DEFER_OK[dev] = False  # frames of this size run in chunks: no deferred first attempt
            raise MatchBudgetExceeded(needed, int(max_scratch))
        cap = int(needed * 1.0625) + 1024
        if max_scratch is not None:
            cap = min(cap, int(max_scratch))
        if cap > _QUERY_CAP.get(dev, 0):
            _QUERY_CAP[dev] = cap
    return offsets, head_off, probes, scanned, total, hcap, ws, nb.value, cap


def query_prefix(index: DeviceIndex, pixels: torch.Tensor, dirs: torch.Tensor, t_near: torch.Tensor,
                 t_far: torch.Tensor, slopes: torch.Tensor, want: int | None = None, footprint: bool = True,
                 max_scratch: int | None = None, whole: int | None = None, sampler_cfg=None) -> QueryPrefix:
    """The query for callers that only want samples (hp_head_count +
    hp_head_sort): each ray's head of matches in (t, id) order, without the
    CSR of all matches."""
    pixels, dirs = pixels.contiguous(), dirs.contiguous()
    return _head(index, _count_head(index, pixels, dirs, t_near, t_far, slopes, footprint, max_scratch), dirs,
                 slopes, want, whole, sampler_cfg)


def count_prefix(index: DeviceIndex, pixels: torch.Tensor, dirs: torch.Tensor, t_near: torch.Tensor,
                 t_far: torch.Tensor, slopes: torch.Tensor, max_scratch: int | None = None) -> QueryPrefix:
    """hp_head_count alone (the count read on the host): a QueryPrefix with
    no heads yet, for :func:`head_resort` over rays that are known to need
    long heads (very dense frames)."""
    pixels, dirs = pixels.contiguous(), dirs.contiguous()
    offsets, head_off, probes, scanned, total, hcap, ws, nb, cap = _count_head(
        index, pixels, dirs, t_near, t_far, slopes, True, max_scratch)
    m = int(offsets.shape[0]) - 1
    pre = QueryPrefix(offsets, probes, scanned, head_off[:m], None, None, None, None, None, None, None, ws, None)
    pre.total = total
    pre.want = pre.whole = HEAD_CAP
    pre._sort_args = (index, dirs, slopes, nb, cap, None)
    return pre


def _head(index, counted, dirs, slopes, want=None, whole=None, sampler_cfg=None) -> QueryPrefix:
    """hp_head_sort after :func:`_count_head` (want / whole default to
    PREFIX_WANT / HEAD_WHOLE, read at call time).  With ``sampler_cfg`` the
    heads carry the sampler's precomputed bound factors."""
    want = PREFIX_WANT if want is None else want
    lib = _lib.load(require_device=True)
    dev = index.row_ptr.device
    offsets, head_off, probes, scanned, total, hcap, ws, nb, cap = counted
    m = int(offsets.shape[0]) - 1
    fa = torch.empty(m, dtype=torch.int32, device=dev)
    plen = torch.empty(m, dtype=torch.int32, device=dev)
    cut = torch.empty((2, m), dtype=torch.float64, device=dev)
    ht = torch.empty(max(hcap, 1), dtype=torch.float64, device=dev)
    hd = torch.empty(max(hcap, 1), dtype=torch.float64, device=dev)
    hi = torch.empty(max(hcap, 1), dtype=torch.int32, device=dev)
    sp = sampler_params(sampler_cfg, False, True) if sampler_cfg is not None else None
    hu = torch.empty(max(hcap, 1), dtype=torch.float32, device=dev) if sp is not None else None
    whole = max(int(want), min(HEAD_WHOLE if whole is None else int(whole), HEAD_CAP))
    _lib.check(lib.hp_head_sort(index.layout(), _ptr(dirs), _ptr(slopes), m, _ptr(offsets), None, 0,
                                _ptr(head_off), int(want), whole, _ptr(ht), _ptr(hi), _ptr(hd), _ptr(plen),
                                _ptr(fa), _ptr(cut[0]), _ptr(cut[1]), ctypes.byref(sp) if sp is not None else None,
                                _ptr(hu), cap, _ptr(ws), nb, _stream()))
    _mark("query.prefix")
    pre = QueryPrefix(offsets, probes, scanned, head_off[:m], plen, ht, hi, hd, cut[0], cut[1], fa, ws, hu)
    pre.total = total
    pre.want, pre.whole = int(want), whole
    pre._sort_args = (index, dirs, slopes, nb, cap, sp)
    return pre


def head_resort(pre: QueryPrefix, rays: torch.Tensor, want: int = HEAD_CAP, whole: int = HEAD_CAP) -> QueryPrefix:
    """Second chance for rays the sampler flagged: re-sort the heads of
    ``rays`` (int64 indices into ``pre``'s rays) from the same count pass
    (``pre`` still holds its workspace) with a longer ``want`` (up to
    HEAD_LONG: ``whole`` > HEAD_CAP is the long-head mode); no re-scan.
    Returns a :class:`QueryPrefix` over just those rays (their own offsets,
    counts unchanged)."""
    lib = _lib.load(require_device=True)
    index, dirs, slopes, nb, cap, sp = pre._sort_args
    dev = pre.offsets.device
    m = int(pre.offsets.shape[0]) - 1
    n = int(rays.numel())
    r32 = rays.to(torch.int32).contiguous()
    counts = (pre.offsets[1:] - pre.offsets[:-1])[rays]
    sub_off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=sub_off[1:])
    whole = max(int(want), min(int(whole), HEAD_LONG))
    per = HEAD_LONG if whole > HEAD_CAP else HEAD_CAP  # head storage per ray
    head_off = torch.arange(n + 1, dtype=torch.int64, device=dev) * per
    fa = torch.empty(n, dtype=torch.int32, device=dev)
    plen = torch.empty(n, dtype=torch.int32, device=dev)
    cut = torch.empty((2, n), dtype=torch.float64, device=dev)
    cap_h = max(n * per, 1)
    ht = torch.empty(cap_h, dtype=torch.float64, device=dev)
    hd = torch.empty(cap_h, dtype=torch.float64, device=dev)
    hi = torch.empty(cap_h, dtype=torch.int32, device=dev)
    hu = torch.empty(cap_h, dtype=torch.float32, device=dev) if sp is not None else None
    _lib.check(lib.hp_head_sort(index.layout(), _ptr(dirs), _ptr(slopes), m, _ptr(pre.offsets), _ptr(r32), n,
                                _ptr(head_off), int(want), whole, _ptr(ht), _ptr(hi), _ptr(hd), _ptr(plen), _ptr(fa),
                                _ptr(cut[0]), _ptr(cut[1]), ctypes.byref(sp) if sp is not None else None, _ptr(hu),
                                cap, _ptr(pre._ws), nb, _stream()))
    sub = QueryPrefix(sub_off, pre.probes[rays], pre.scanned[rays], head_off[:n], plen, ht, hi, hd, cut[0], cut[1],
                      fa, pre._ws, hu)
    sub.total = None
    sub.want, sub.whole = int(want), whole
    sub._sort_args = None
    return sub


def query_frame(index: DeviceIndex, pixels, dirs, t_near, t_far, slopes, prefix: bool | None = None,
                max_scratch: int | None = None, want: int | None = None, sampler_cfg=None, defer=None):
    """The query of a sampling frame: the heads (``prefix`` True or None;
    returns a :class:`QueryPrefix`) or the full CSR with facts (``prefix``
    False; returns the 7-tuple of :func:`query`).  ``defer`` (None:
    DEFER_COUNT): no host read after the head count (sample_prefix then
    checks it and raises :class:`CountShort` when it ran short)."""
    pixels, dirs = pixels.contiguous(), dirs.contiguous()
    if prefix is False:
        return _fill(index, _count(index, pixels, dirs, t_near, t_far, slopes, True, max_scratch), slopes, True)
    defer = DEFER_COUNT if defer is None else defer
    return _head(index, _count_head(index, pixels, dirs, t_near, t_far, slopes, True, max_scratch, defer, True),
                 dirs, slopes, want, None, sampler_cfg)


def sampler_params(cfg, want_color: bool, exact_t_end: bool, emit_knn: bool = False) -> _lib.SamplerParams:
    """C parameter block from a SamplerConfig; a ready _lib.SamplerParams
    (the reference operator's raw arguments, e.g. beta2 given directly) is
    taken as is, with want_color / exact_t_end applied."""
    if isinstance(cfg, _lib.SamplerParams):
        p = _lib.SamplerParams()
        ctypes.pointer(p)[0] = cfg
        p.want_color = 1 if want_color else 0
        p.exact_t_end = 1 if exact_t_end else 0
        p.emit_knn = 1 if emit_knn else 0
        return p
    p = _lib.SamplerParams()
    p.emit_knn = 1 if emit_knn else 0
    p.k_neighbors = int(cfg.k_neighbors)
    p.eps_mode = 1 if cfg.retention_mode == "epsilon" else 0
    p.want_color = 1 if want_color else 0
    p.exact_t_end = 1 if exact_t_end else 0
    p.beta2 = float(cfg.beta * cfg.beta)      # as sampler.py:215
    p.gamma = float(cfg.gamma)
    p.eps = float(cfg.epsilon)
    p.tau_min = float(cfg.tau_min)
    return p


def sample(offsets: torch.Tensor, ids: torch.Tensor, t: torch.Tensor, dist: torch.Tensor,
           slopes: torch.Tensor, cfg, colors: torch.Tensor | None = None,
           exact_t_end: bool = True, facts: torch.Tensor | None = None, emit_knn: bool = False):
    """_kernels.sample_batch on the device (reference _kernels.py:552-700).

    Returns (r_off, r_id, r_t, r_dist, r_udf, r_alpha, r_w, r_color, t_end).
    ``exact_t_end=False`` stops each ray once retention is decided and reports
    the transmittance at that point instead of over all candidates.
    ``facts``: the per-ray facts :func:`query` returned with this very CSR and
    these slopes (lets the sampler skip its full precondition pass); results
    are identical with or without them.  ``emit_knn``: two more outputs, the
    retained samples' K neighbour point ids (int64 [R, K], -1 past the pool)
    and blend weights (float64 [R, K]) -- north_star stage 4's per-sample
    candidate indices and weights (the K nearest of _kernels.py:603-620).
    """
    lib = _lib.load(require_device=True)
    dev = offsets.device
    m = int(offsets.shape[0]) - 1
    total = int(ids.numel())
    want = colors is not None
    p = sampler_params(cfg, want, exact_t_end, emit_knn)
    exact_cap = max(SAMPLE_EXACT_PER_RAY * m, 1 << 16)
    r_off = torch.empty(m + 1, dtype=torch.int64, device=dev)
    t_end = torch.empty(max(m, 0), dtype=torch.float64, device=dev)
    col = colors.contiguous() if want else None
    ncol = int(col.shape[0]) if want else 0
    _mark("sample.setup")
    for _ in range(2):
        nb = c_size(0)
        _lib.check(lib.hp_sample_workspace_bytes(m, total, exact_cap, ctypes.byref(p),
                                                 ctypes.byref(nb)))
        ws = _workspace(nb.value, dev)
        common = (_ptr(offsets), m, _ptr(ids), _ptr(t), _ptr(dist), total, exact_cap,
                  _ptr(slopes), ctypes.byref(p), _ptr(col) if want else ctypes.c_void_p(0), ncol)
        run_args = common[:8] + (_ptr(facts) if facts is not None else ctypes.c_void_p(0),) + common[8:]
        _lib.check(lib.hp_sample_run(*run_args, _ptr(r_off), _ptr(t_end), _ptr(ws), nb.value, _stream()))
        _mark("sample.run")
        R = _host_read(r_off[m])[0]
        if R >= 0:
            break
        exact_cap = int(-R * 1.0625) + 1024   # exact scratch too small: grow it once
    i64 = dict(dtype=torch.int64, device=dev)
    f64 = dict(dtype=torch.float64, device=dev)
    r_id = torch.empty(R, **i64)
    outs = [torch.empty(R, **f64) for _ in range(5)]
    r_color = torch.empty((R, 3), **f64) if want else torch.zeros((0, 3), **f64)
    knn = _knn_outputs(R, p, dev)
    _mark("sample.sync")
    _lib.check(lib.hp_sample_emit(*common, _ptr(r_off), R, _ptr(r_id), *[_ptr(o) for o in outs],
                                  _ptr(r_color) if want else ctypes.c_void_p(0), *_knn_ptrs(knn), _ptr(ws),
                                  nb.value, _stream()))
    _mark("sample.emit")
    return (r_off, r_id, *outs, r_color, t_end, *knn)


def _knn_ptrs(knn):
    return [_ptr(x) for x in knn] if knn else [ctypes.c_void_p(0), ctypes.c_void_p(0)]


def _knn_outputs(R, p, dev):
    if not p.emit_knn:
        return ()
    return (torch.empty((R, p.k_neighbors), dtype=torch.int64, device=dev),
            torch.empty((R, p.k_neighbors), dtype=torch.float64, device=dev))


def sample_prefix(pre: QueryPrefix, slopes: torch.Tensor, cfg, colors: torch.Tensor | None = None,
                  exact_t_end: bool = False, emit_knn: bool = False):
    """:func:`sample` over :func:`query_prefix`'s prefixes
    (hp_sample_run_prefix / hp_sample_emit_prefix).

    Returns (r_off, r_id, r_t, r_dist, r_udf, r_alpha, r_w, r_color, t_end,
    flagged, n_flagged): for every ray with ``flagged[r] == 0`` the results
    are :func:`sample`'s on the full CSR; a flagged ray (its work may reach
    past its prefix) has no retained candidates and t_end NaN here and must
    be run through the full path (:func:`sample_rays_prefix` does that).
    """
    lib = _lib.load(require_device=True)
    dev = pre.offsets.device
    m = int(pre.offsets.shape[0]) - 1
    want = colors is not None
    p = sampler_params(cfg, want, exact_t_end, emit_knn)
    exact_cap = max(SAMPLE_EXACT_PER_RAY * m, 1 << 16)
    r_off = torch.empty(m + 1, dtype=torch.int64, device=dev)
    t_end = torch.empty(max(m, 0), dtype=torch.float64, device=dev)
    flagged = torch.empty(m + 1, dtype=torch.int32, device=dev)
    col = colors.contiguous() if want else None
    ncol = int(col.shape[0]) if want else 0
    sp = pre.struct()
    colp = _ptr(col) if want else ctypes.c_void_p(0)
    for _ in range(2):
        nb = c_size(0)
        _lib.check(lib.hp_sample_workspace_bytes(m, 0, exact_cap, ctypes.byref(p), ctypes.byref(nb)))
        ws = _workspace(nb.value, dev)
        _lib.check(lib.hp_sample_run_prefix(_ptr(pre.offsets), m, ctypes.byref(sp), exact_cap, _ptr(slopes),
                                            _ptr(pre.facts), ctypes.byref(p), colp, ncol, _ptr(r_off),
                                            _ptr(t_end), _ptr(flagged), _ptr(ws), nb.value, _stream()))
        _mark("sample.run")
        vals = [r_off[m], flagged[m].to(torch.int64)]
        if pre.total is None:  # deferred count: Q (or a short count) read here too
            vals.append(pre.offsets[m])
        both = _host_read(*vals)  # one synchronisation
        R, n_flagged = both[0], both[1]
        if pre.total is None:
            pre.total = int(both[2])
            if pre.total < 0:
                _DEFER_OK[dev] = False
                raise CountShort(-pre.total)
        if R >= 0:
            break
        exact_cap = int(-R * 1.0625) + 1024   # exact scratch too small: grow it once
    i64 = dict(dtype=torch.int64, device=dev)
    f64 = dict(dtype=torch.float64, device=dev)
    r_id = torch.empty(R, **i64)
    outs = [torch.empty(R, **f64) for _ in range(5)]
    r_color = torch.empty((R, 3), **f64) if want else torch.zeros((0, 3), **f64)
    knn = _knn_outputs(R, p, dev)
    _lib.check(lib.hp_sample_emit_prefix(_ptr(pre.offsets), m, ctypes.byref(sp), exact_cap, _ptr(slopes),
                                         ctypes.byref(p), colp, ncol, _ptr(r_off), R, _ptr(r_id),
                                         *[_ptr(o) for o in outs], _ptr(r_color) if want else ctypes.c_void_p(0),
                                         *_knn_ptrs(knn), _ptr(ws), nb.value, _stream()))
    _mark("sample.emit")
    return (r_off, r_id, *outs, r_color, t_end, *knn, flagged[:m], n_flagged)


def merge_flagged(main, flagged: torch.Tensor, sub, sel: torch.Tensor | None = None):
    """Splice the full-path samples ``sub`` of the flagged rays into the
    prefix-mode samples ``main`` (both (r_off, r_id, r_t, r_dist, r_udf,
    r_alpha, r_w, r_color, t_end[, r_knn_id, r_knn_w])); flagged rays hold no
    candidates in main.  ``sel``: the flagged ray indices if the caller has
    them already.  One copy kernel (hp_splice_samples)."""
    lib = _lib.load(require_device=True)
    r_off, s_off = main[0], sub[0]
    dev = r_off.device
    m = int(r_off.shape[0]) - 1
    if sel is None:
        sel = torch.nonzero(flagged, as_tuple=True)[0]
    counts = r_off[1:] - r_off[:-1]
    counts[sel] = s_off[1:] - s_off[:-1]
    off = torch.zeros(m + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=off[1:])
    R_main, R_sub = int(main[1].shape[0]), int(sub[1].shape[0])  # host values: no synchronisation
    R = R_main + R_sub  # flagged rays hold nothing in main
    pos = torch.full((m,), -1, dtype=torch.int64, device=dev)
    pos[sel] = torch.arange(int(sel.numel()), dtype=torch.int64, device=dev)
    colours = main[7].shape[0] == R_main and sub[7].shape[0] == R_sub and (R_main + R_sub == 0 or
                                                                            main[7].numel() + sub[7].numel() > 0)
    knn = len(main) > 9
    K = int(main[9].shape[1]) if knn else 0
    out = [off, torch.empty(R, dtype=torch.int64, device=dev)] + \
        [torch.empty(R, dtype=torch.float64, device=dev) for _ in range(5)]
    out.append(torch.empty((R, 3), dtype=torch.float64, device=dev) if colours
               else torch.zeros((0, 3), dtype=torch.float64, device=dev))
    te = main[8].clone()
    te[sel] = sub[8]
    out.append(te)
    if knn:
        out += [torch.empty((R, K), dtype=torch.int64, device=dev), torch.empty((R, K), dtype=torch.float64,
                                                                                device=dev)]

    def fields(t):
        f = _lib.SampleFields(*[t[k].data_ptr() if t[k].numel() else 0 for k in range(1, 7)])
        f.r_color = t[7].data_ptr() if (colours and t[7].numel()) else None
        if knn:
            f.r_knn_id, f.r_knn_w = (t[9].data_ptr() or None), (t[10].data_ptr() or None)
        return f
    if R:
        A, B, O = fields(main), fields(sub), fields(out)
        _lib.check(lib.hp_splice_samples(m, _ptr(off), _ptr(r_off), _ptr(s_off), _ptr(pos), K, ctypes.byref(A),
                                         ctypes.byref(B), ctypes.byref(O), _stream()))
    return tuple(out)


def ray_grid(camera, dev=None, row0: int = 0, rows: int | None = None, t_near: float | None = None,
             t_far: float | None = None):
    """geometry.ray_grid on the device (hp_ray_grid, bit-identical to numpy;
    reference geometry.py:289-306): (dirs f64 [m,3], pixels i64 [m,2]) for
    image rows [row0, row0 + rows), plus t_near / t_far [m] filled with the
    given scalars (None when not given)."""
    lib = _lib.load(require_device=True)
    dev = dev or torch.device("cuda", torch.cuda.current_device())
    rows = int(camera.height) - row0 if rows is None else int(rows)
    m = rows * int(camera.width)
    dirs = torch.empty((m, 3), dtype=torch.float64, device=dev)
    pixels = torch.empty((m, 2), dtype=torch.int64, device=dev)
    tn = torch.empty(m, dtype=torch.float64, device=dev) if t_near is not None else None
    tf = torch.empty(m, dtype=torch.float64, device=dev) if t_far is not None else None
    _lib.check(lib.hp_ray_grid(ctypes.byref(camera_struct(camera)), int(row0), rows, _ptr(dirs), _ptr(pixels),
                               float(t_near or 0.0), float(t_far or 0.0),
                               _ptr(tn) if tn is not None else ctypes.c_void_p(0),
                               _ptr(tf) if tf is not None else ctypes.c_void_p(0), _stream()))
    return dirs, pixels, tn, tf


def radius_slopes(camera, kernel_radius: float, approx: bool = False, pixels: torch.Tensor | None = None,
                  row0: int = 0, m: int | None = None, dev=None) -> torch.Tensor:
    """geometry.radius_slopes on the device (hp_radius_slopes, bit-identical
    to numpy; reference geometry.py:249-260): for ``pixels`` (int64 [m, 2] on
    the device), or for rays row0 * W .. row0 * W + m of the camera's ray grid."""
    lib = _lib.load(require_device=True)
    if pixels is not None:
        if pixels.stride(-1) != 1:
            pixels = pixels.contiguous()
        dev = pixels.device
        m = int(pixels.shape[0])
        stride = int(pixels.stride(0)) if m else 2
    else:
        dev = dev or torch.device("cuda", torch.cuda.current_device())
        m = int(camera.width) * int(camera.height) - row0 * int(camera.width) if m is None else int(m)
        stride = 2
    out = torch.empty(m, dtype=torch.float64, device=dev)
    _lib.check(lib.hp_radius_slopes(ctypes.byref(camera_struct(camera)), int(row0),
                                    _ptr(pixels) if pixels is not None else ctypes.c_void_p(0), stride, m,
                                    float(kernel_radius), 1 if approx else 0, _ptr(out), _stream()))
    return out


def primary_surface(r_off: torch.Tensor, r_id: torch.Tensor, r_t: torch.Tensor):
    """Primary-surface point per ray: (point id or -1, t or NaN)."""
    lib = _lib.load(require_device=True)
    m = int(r_off.shape[0]) - 1
    pid = torch.empty(m, dtype=torch.int64, device=r_off.device)
    pt = torch.empty(m, dtype=torch.float64, device=r_off.device)
    _lib.check(lib.hp_primary_surface(_ptr(r_off), m, _ptr(r_id), _ptr(r_t), _ptr(pid),
                                      _ptr(pt), _stream()))
    return pid, pt
