"""Chained search -> sampling, the way the reference's renderer drives the path
(renderer._prepare, reference renderer.py:113-125: query_batch_arrays then
sample_batch_arrays on the same CSR).

Here the query CSR never leaves HBM: only rays/points go up and the retained
samples come back.  ``frame_device`` is the all-device step the benchmark
times; ``search_and_sample`` is the host-buffer public entry point (numpy in,
numpy out) used for the end-to-end number.
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import device
from .sampler import SamplerConfig

__all__ = ["FrameResult", "frame_device", "search_and_sample", "search_and_sample_view",
           "search_and_sample_views", "StageTimer", "host_slopes"]


SLOPE_THREADS = int(os.environ.get("HP_SLOPE_THREADS", "0")) or min(16, os.cpu_count() or 1)
H2D_THREADS = int(os.environ.get("HP_H2D_THREADS", "0")) or min(4, os.cpu_count() or 1)
# pageable uploads through hp_host_upload (host threads + pinned staging) instead of the driver's own path
H2D_STAGED = os.environ.get("HP_H2D_STAGED", "1") == "1"


def host_slopes(camera, pixels: np.ndarray | None, kernel_radius: float, approx: bool = False,
                out: np.ndarray | None = None, threads: int | None = None) -> np.ndarray:
    """``radius_slopes`` on host threads through the library
    (hp_radius_slopes_host: same expression order and libm calls as numpy,
    bit-identical).  ``pixels=None``: the camera's whole ray grid (row-major,
    as ``ray_grid``).  ``out`` may be a (pinned) float64 buffer of m values."""
    lib = device._lib.load(require_device=False)
    if pixels is None:
        px, m = None, int(camera.width) * int(camera.height)
    else:
        px = np.ascontiguousarray(pixels, dtype=np.int64).reshape(-1, 2)
        m = px.shape[0]
    if out is None:
        out = np.empty(m, dtype=np.float64)
    threads = threads or SLOPE_THREADS
    device._lib.check(lib.hp_radius_slopes_host(ctypes.byref(device.camera_struct(camera)),
                                                px.ctypes.data_as(ctypes.c_void_p) if px is not None
                                                else ctypes.c_void_p(0), 2, m,
                                                float(kernel_radius), 1 if approx else 0,
                                                out.ctypes.data_as(ctypes.c_void_p), int(threads)))
    return out


class StageTimer:
    """CUDA-event timer around the C-ABI calls of one frame (on the stream the
    kernels are launched on, i.e. torch's current stream)."""

    def __init__(self):
        self.events = []

    def mark(self, name):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.append((name, ev))

    def spans(self) -> dict:
        torch.cuda.synchronize()
        out = {}
        for (a, ea), (b, eb) in zip(self.events[:-1], self.events[1:]):
            out[b] = out.get(b, 0.0) + ea.elapsed_time(eb)
        return out


@dataclass
class FrameResult:
    index: device.DeviceIndex
    query: tuple | None      # the query CSR (None when the frame ran in ray chunks)
    samples: tuple
    Q: int = 0
    chunks: int = 1
    flagged: int = 0         # prefix mode: rays re-run through the full query
    resorted: int = 0        # prefix mode: rays whose heads were re-sorted longer (second chance)
    prefix: bool = False     # the frame ran in prefix mode
    prefix_len: object = None  # TRACK_PREFIX_LEN: device int64[4] (Σ head length, Σ q cut / whole, hit rays)

    @property
    def R(self) -> int:
        return int(self.samples[1].numel())


# bytes of device memory per match slot of one query + sample pass, for
# sizing ray chunks: unsorted scratch 20 + CSR 24 + sampler scratch (bounded);
# head mode: (key, slot) scratch 8 + at most one 20-byte head entry
BYTES_PER_MATCH = 56
BYTES_PER_MATCH_PREFIX = 28


_BUDGET: dict = {}
_SIDE: dict = {}


def _side_stream(dev) -> torch.cuda.Stream:
    if dev not in _SIDE:
        _SIDE[dev] = torch.cuda.Stream(device=dev)
    return _SIDE[dev]


def match_budget(fraction: float = 0.8, bytes_per_match: int = BYTES_PER_MATCH) -> int:
    """Match slots one pass may use: a fraction of the device memory free at
    the first call (cached per device: cudaMemGetInfo costs milliseconds)."""
    dev = torch.cuda.current_device()
    if dev not in _BUDGET:
        free, _ = torch.cuda.mem_get_info()
        free += torch.cuda.memory_reserved() - torch.cuda.memory_allocated()  # torch's cached blocks
        _BUDGET[dev] = int(free * fraction)
    return max(_BUDGET[dev] // bytes_per_match, 1 << 20)


def _concat_samples(parts):
    """Concatenate per-chunk sampler 9-tuples (offsets rebased)."""
    if len(parts) == 1:
        return parts[0]
    offs, base = [parts[0][0][:1]], 0
    for p in parts:
        offs.append(p[0][1:] + base)
        base += int(p[1].numel())
    out = [torch.cat(offs)]
    for k in range(1, len(parts[0])):
        out.append(torch.cat([p[k] for p in parts]))
    return tuple(out)


def frame_device(xyz: torch.Tensor, colors: torch.Tensor | None, camera, search_cfg, pixels,
                 dirs, t_near, t_far, slopes, sampler_cfg: SamplerConfig | None = None,
                 exact_t_end: bool = True, timer: StageTimer | None = None,
                 max_matches: int | None = None, emit_knn: bool = False,
                 rows: tuple | None = None) -> FrameResult:
    """build -> query -> sample, all on the device (CUDA tensors in and out).

    A frame whose query would need more than ``max_matches`` match slots
    (default: :func:`match_budget`) runs in ray chunks (ray-chunk
    streaming): the per-ray bounds split the rays, each chunk is queried and
    sampled in turn, and only the retained samples are kept.  Results are
    identical (rays are independent).  The index is the query layout alone
    (device.build_layout: no reference HashIndex arrays); ``rows`` = (a, b)
    when every ray lies in image rows [a, b) (a row band): only the points
    those rays can reach are placed."""
    mark = timer.mark if timer is not None else (lambda name: None)
    mark("start")
    idx = device.build_layout(xyz, camera, search_cfg.pad, rows)
    mark("build")
    return _query_sample(idx, colors, pixels, dirs, t_near, t_far, slopes, sampler_cfg or SamplerConfig(),
                         exact_t_end, max_matches, mark, emit_knn=emit_knn)


# Frames that only want samples keep 8 bytes per match and sort each ray's
# head only (device.query_prefix = hp_head_count + hp_head_sort, then
# device.sample_prefix: no query CSR); rays whose sampling may reach past the
# head re-run through the full query.  HP_PREFIX=0 uses the full CSR.
_PREFIX_ENV = os.environ.get("HP_PREFIX", "1")
PREFIX = _PREFIX_ENV != "0"


_PREFIX_LEN: list = []  # head statistics of the passes of the current frame (device tensors)
TRACK_PREFIX_LEN = False  # bench.py: report the head statistics (a few extra reductions per pass)
FLAG_REASONS: list = []  # with TRACK_PREFIX_LEN: per pass, counts of flagged rays by reason 1..5


def _prefix_finish(pre, idx, colors, pixels, dirs, t_near, t_far, slopes, sampler_cfg, exact_t_end, budget=None,
                   emit_knn=False):
    """Sample over the heads of ``pre``.  Rays whose sampling may reach past
    their head get a second chance: their heads are re-sorted from the same
    count pass up to 1024 matches (device.head_resort, no re-scan) and
    sampled again; the few still flagged re-run through the full query (within
    ``budget`` full-path match slots -- default: from the free memory -- in
    ray chunks when they need more).  (samples 9-tuple, Q, rays re-run on the
    full path, rays re-sorted)"""
    *s, flagged, n_flagged = device.sample_prefix(pre, slopes, sampler_cfg, colors, exact_t_end, emit_knn)
    Q = pre.total
    if TRACK_PREFIX_LEN:  # flag reasons (hp_sample.cu plan_ray) of this pass
        FLAG_REASONS.append(torch.bincount(flagged.to(torch.int64), minlength=6)[1:6])
    if TRACK_PREFIX_LEN:  # [Σ head length, Σ q of the cut rays, Σ q of the whole rays, rays with matches]
        q = pre.offsets[1:] - pre.offsets[:-1]
        cut = q > pre.whole
        _PREFIX_LEN.append(torch.stack([pre.length.sum().to(torch.int64), torch.where(cut, q, 0).sum(),
                                        torch.where(cut, 0, q).sum(), (q > 0).sum()]))
    n_full, n_resorted = 0, 0
    if n_flagged:
        sel = torch.nonzero(flagged, as_tuple=True)[0]
        m = int(pre.offsets.shape[0]) - 1
        direct = False
        if LONG_HEADS and n_flagged > LONG_DIRECT * m:
            # many rays flagged, most of them far longer than 1024 matches (very
            # dense rays): a 1024-entry second chance would mostly fail
            q_sel = (pre.offsets[1:] - pre.offsets[:-1])[sel]
            direct = int((q_sel > 2 * device.HEAD_CAP).sum()) > n_flagged // 2
        if direct:
            n_resorted = n_flagged
            pre.t = pre.ids = pre.dist = None
            sub, n_full = _long_heads(pre, idx, colors, pixels, dirs, t_near, t_far, slopes, sel, sampler_cfg,
                                      exact_t_end, budget, emit_knn)
            s = device.merge_flagged(tuple(s), flagged, sub, sel)
        elif pre.want < device.HEAD_CAP:  # second chance: longer heads from the same count pass
            n_resorted = n_flagged
            sub_pre = device.head_resort(pre, sel)
            pre.t = pre.ids = pre.dist = None  # (the count pass's workspace stays for a third chance)
            sl = slopes[sel]
            *s2, fl2, nf2 = device.sample_prefix(sub_pre, sl, sampler_cfg, colors, exact_t_end, emit_knn)
            sub_pre.t = sub_pre.ids = sub_pre.dist = sub_pre._ws = None
            if nf2:
                sel2 = torch.nonzero(fl2, as_tuple=True)[0]
                r2 = sel[sel2]
                if LONG_HEADS:  # third chance: heads of up to HEAD_LONG, still from the count pass
                    sub2, n_full = _long_heads(pre, idx, colors, pixels, dirs, t_near, t_far, slopes, r2,
                                               sampler_cfg, exact_t_end, budget, emit_knn)
                else:
                    sub2 = _full_rays(idx, colors, pixels[r2], dirs[r2], t_near[r2], t_far[r2], slopes[r2],
                                      sampler_cfg, exact_t_end, budget, emit_knn)
                    n_full = nf2
                s2 = device.merge_flagged(tuple(s2), fl2, sub2, sel2)
            s = device.merge_flagged(tuple(s), flagged, tuple(s2), sel)
        elif LONG_HEADS and pre.want < device.HEAD_LONG:  # heads already 1024 long: the long heads next
            n_resorted = n_flagged
            pre.t = pre.ids = pre.dist = None
            sub, n_full = _long_heads(pre, idx, colors, pixels, dirs, t_near, t_far, slopes, sel, sampler_cfg,
                                      exact_t_end, budget, emit_knn)
            s = device.merge_flagged(tuple(s), flagged, sub, sel)
        else:
            pre.t = pre.ids = pre.dist = pre._ws = None
            sub = _full_rays(idx, colors, pixels[sel], dirs[sel], t_near[sel], t_far[sel], slopes[sel], sampler_cfg,
                             exact_t_end, budget, emit_knn)
            s = device.merge_flagged(tuple(s), flagged, sub, sel)
            n_full = n_flagged
    # the heads and their workspace are no longer needed (sample_prefix copied its outputs)
    pre.t = pre.ids = pre.dist = pre._ws = None
    return tuple(s), Q, n_full, n_resorted


# rays the 1024-entry second chance leaves flagged get heads of up to
# device.HEAD_LONG (HP_LONG_HEADS=0: straight to the full query), in batches
# of at most LONG_BATCH rays (24 bytes of head storage per entry)
LONG_HEADS = os.environ.get("HP_LONG_HEADS", "1") == "1"
LONG_BATCH = int(os.environ.get("HP_LONG_BATCH", str(1 << 15)))
LONG_DIRECT = float(os.environ.get("HP_LONG_DIRECT", "0.25"))  # flagged fraction that skips the 1024 heads
# ray chunks whose footprint bound exceeds this many slots per ray start with the long heads
LONG_FIRST = int(os.environ.get("HP_LONG_FIRST", "16384"))


def _long_heads(pre, idx, colors, pixels, dirs, t_near, t_far, slopes, rays, sampler_cfg, exact_t_end, budget,
                emit_knn=False):
    """Samples of ``rays`` (indices into ``pre``'s rays) over heads of up to
    device.HEAD_LONG re-sorted from ``pre``'s count pass; the rays still
    flagged take the full query.  (samples of ``rays`` in order, rays on the
    full path)"""
    parts, n_full = [], 0
    for a in range(0, int(rays.numel()), LONG_BATCH):
        r = rays[a:a + LONG_BATCH]
        sub = device.head_resort(pre, r, want=device.HEAD_LONG, whole=device.HEAD_LONG)
        *s3, fl3, nf3 = device.sample_prefix(sub, slopes[r], sampler_cfg, colors, exact_t_end, emit_knn)
        sub.t = sub.ids = sub.dist = sub._ws = None
        if nf3:
            sel3 = torch.nonzero(fl3, as_tuple=True)[0]
            r3 = r[sel3]
            full = _full_rays(idx, colors, pixels[r3], dirs[r3], t_near[r3], t_far[r3], slopes[r3], sampler_cfg,
                              exact_t_end, budget, emit_knn)
            s3 = device.merge_flagged(tuple(s3), fl3, full, sel3)
            n_full += nf3
        parts.append(tuple(s3))
    return _concat_samples(parts), n_full


def _full_rays(idx, colors, pixels, dirs, t_near, t_far, slopes, sampler_cfg, exact_t_end, budget, emit_knn=False):
    """Full-CSR query + sample of a set of rays, in ray chunks of at most
    ``budget`` match slots."""
    if budget is None:
        budget = match_budget(bytes_per_match=BYTES_PER_MATCH)
    try:
        q = device.query(idx, pixels, dirs, t_near, t_far, slopes, facts=True, max_scratch=budget)
    except device.MatchBudgetExceeded:
        return _frame_chunked(idx, colors, pixels, dirs, t_near, t_far, slopes, sampler_cfg, exact_t_end, budget,
                              lambda name: None, prefix=False, emit_knn=emit_knn).samples
    s = device.sample(q[0], q[1], q[2], q[3], slopes, sampler_cfg, colors, exact_t_end, facts=q[6],
                      emit_knn=emit_knn)
    del q
    return s


def _prefix_pass(idx, colors, pixels, dirs, t_near, t_far, slopes, sampler_cfg, exact_t_end, budget=None,
                 emit_knn=False, long_first=False):
    if long_first and LONG_HEADS:  # very dense rays: the long heads from the start
        pre = device.count_prefix(idx, pixels, dirs, t_near, t_far, slopes)
        m = int(pre.offsets.shape[0]) - 1
        s, n_full = _long_heads(pre, idx, colors, pixels, dirs, t_near, t_far, slopes,
                                torch.arange(m, device=pre.offsets.device), sampler_cfg, exact_t_end, budget,
                                emit_knn)
        pre._ws = None
        return s, int(pre.total), n_full, m
    pre = device.query_prefix(idx, pixels, dirs, t_near, t_far, slopes,
                              sampler_cfg=sampler_cfg if device.HEAD_FACTORS else None)
    return _prefix_finish(pre, idx, colors, pixels, dirs, t_near, t_far, slopes, sampler_cfg, exact_t_end, budget,
                          emit_knn)


def _query_sample(idx, colors, pixels, dirs, t_near, t_far, slopes, sampler_cfg, exact_t_end, max_matches,
                  mark=lambda name: None, before_sample=lambda: None, prefix: bool | None = None,
                  emit_knn: bool = False) -> FrameResult:
    """query -> sample of one frame on the device.  ``prefix``: True (heads)
    / False (full CSR); None: the HP_PREFIX setting.  ``colors`` may be a
    callable that returns them (called once the query is enqueued)."""
    prefix = PREFIX if prefix is None else prefix
    budget = int(max_matches) if max_matches is not None else match_budget(
        bytes_per_match=BYTES_PER_MATCH_PREFIX if prefix else BYTES_PER_MATCH)
    col = []

    def colours():
        if not col:
            col.append(colors() if callable(colors) else colors)
        return col[0]
    try:
        return _query_sample_once(idx, colours, pixels, dirs, t_near, t_far, slopes, sampler_cfg, exact_t_end,
                                  max_matches, mark, before_sample, prefix, emit_knn, budget, None)
    except device.CountShort:  # the deferred count ran short: again, reading the count first
        return _query_sample_once(idx, colours, pixels, dirs, t_near, t_far, slopes, sampler_cfg, exact_t_end,
                                  max_matches, mark, lambda: None, prefix, emit_knn, budget, False)


def _query_sample_once(idx, colours, pixels, dirs, t_near, t_far, slopes, sampler_cfg, exact_t_end, max_matches,
                       mark, before_sample, prefix, emit_knn, budget, defer) -> FrameResult:
    try:
        q = device.query_frame(idx, pixels, dirs, t_near, t_far, slopes, prefix=prefix, max_scratch=budget,
                               sampler_cfg=sampler_cfg if device.HEAD_FACTORS else None, defer=defer)
    except device.MatchBudgetExceeded:
        # too big for one pass: ray chunks (prefix mode unless turned off --
        # such frames are dominated by long rays)
        before_sample()
        return _frame_chunked(idx, colours(), pixels, dirs, t_near, t_far, slopes, sampler_cfg,
                              exact_t_end, budget, mark, prefix is not False, max_matches, emit_knn)
    mark("query")
    before_sample()
    colors = colours()
    if isinstance(q, device.QueryPrefix):
        _PREFIX_LEN.clear()
        s, Q, n_flagged, n_res = _prefix_finish(q, idx, colors, pixels, dirs, t_near, t_far, slopes, sampler_cfg,
                                                exact_t_end, max_matches, emit_knn)
        mark("sample")
        return FrameResult(idx, None, s, Q=Q, flagged=n_flagged, resorted=n_res, prefix=True,
                           prefix_len=_PREFIX_LEN.pop() if _PREFIX_LEN else None)
    s = device.sample(q[0], q[1], q[2], q[3], slopes, sampler_cfg, colors, exact_t_end, facts=q[6],
                      emit_knn=emit_knn)
    mark("sample")
    return FrameResult(idx, q[:6], s, Q=int(q[1].numel()))


def _frame_chunked(idx, colors, pixels, dirs, t_near, t_far, slopes, sampler_cfg, exact_t_end,
                   budget, mark, prefix=False, rerun_budget=None, emit_knn=False):
    bo = device.query_bounds(idx, pixels, dirs, t_near, t_far, slopes).cpu().numpy()
    m = bo.shape[0] - 1
    cuts = [0]
    while cuts[-1] < m:
        a = cuts[-1]
        b = int(np.searchsorted(bo, bo[a] + budget, side="right")) - 1
        if b <= a:
            raise device.MatchBudgetExceeded(int(bo[a + 1] - bo[a]), budget)
        cuts.append(min(b, m))
    # every chunk's scratch need is below its bound: size the counts for the
    # largest chunk up front (a count over a short capacity wastes a pass)
    dev = idx.device
    big = max(int(bo[b] - bo[a]) for a, b in zip(cuts[:-1], cuts[1:]))
    device._QUERY_CAP[dev] = max(device._QUERY_CAP.get(dev, 0), big)
    parts, Q, nf, nr = [], 0, 0, 0
    _PREFIX_LEN.clear()
    for a, b in zip(cuts[:-1], cuts[1:]):
        if prefix:
            dense = (bo[b] - bo[a]) > LONG_FIRST * (b - a)  # the rays' footprint slots bound their matches
            s, q_n, f_n, r_n = _prefix_pass(idx, colors, pixels[a:b], dirs[a:b], t_near[a:b], t_far[a:b],
                                            slopes[a:b], sampler_cfg, exact_t_end, rerun_budget, emit_knn,
                                            long_first=dense)
            parts.append(s)
            Q += q_n
            nf += f_n
            nr += r_n
            continue
        q = device.query(idx, pixels[a:b], dirs[a:b], t_near[a:b], t_far[a:b], slopes[a:b], facts=True)
        parts.append(device.sample(q[0], q[1], q[2], q[3], slopes[a:b], sampler_cfg, colors,
                                   exact_t_end, facts=q[6], emit_knn=emit_knn))
        Q += int(q[1].numel())
        del q
    mark("query")
    mark("sample")
    plen = sum(_PREFIX_LEN) if (prefix and _PREFIX_LEN) else None
    _PREFIX_LEN.clear()
    return FrameResult(idx, None, _concat_samples(parts), Q=Q, chunks=len(parts), flagged=nf, resorted=nr,
                       prefix=prefix, prefix_len=plen)


# Host-buffer calls run the frame in ray chunks so that the result copies
# overlap the device work: every chunk's samples go down (pinned buffers, a
# copy stream) while the next one computes, and only the last, smaller
# chunk's copy is exposed.  Each extra chunk costs ~0.4 ms of device time
# (cfg2), so one cut.  Rays are independent: the samples are one pass's.
_CUTS_ENV = os.environ.get("HP_E2E_CUTS", "0.6")
E2E_CUTS = tuple(float(x) for x in _CUTS_ENV.split(",") if x.strip()) if _CUTS_ENV != "none" else ()
E2E_MIN_RAYS = 1 << 17   # smaller frames: one pass
E2E_HEADROOM = 1.25      # host buffers: the first chunk's sample density times this
_R_PER_RAY: dict = {}    # last frame's samples per ray, per device: the host buffers' first size
_COPY: dict = {}


def _copy_stream(dev) -> torch.cuda.Stream:
    if dev not in _COPY:
        _COPY[dev] = torch.cuda.Stream(device=dev)
    return _COPY[dev]


def _ray_chunks(m: int) -> list:
    if m < E2E_MIN_RAYS or not E2E_CUTS:
        return [0, m]
    cuts = sorted({0, m, *(min(max(int(f * m), 0), m) for f in E2E_CUTS)})
    return cuts


def _host_buffers(s, m, cap, old=None, rows=0):
    """Pinned host buffers for a frame's samples: offsets [m + 1], t_end [m]
    and the per-sample fields with room for ``cap`` samples (the first
    ``rows`` of ``old`` carried over when growing)."""
    R = int(s[1].shape[0])
    out = []
    for k, x in enumerate(s):
        if k in (0, 8):
            out.append(old[k] if old is not None else
                       torch.empty(m + 1 if k == 0 else m, dtype=x.dtype, pin_memory=True))
        elif x.shape[0] != R:  # no colours: (0, 3)
            out.append(torch.zeros(tuple(x.shape), dtype=x.dtype))
        else:
            h = torch.empty((cap,) + tuple(x.shape[1:]), dtype=x.dtype, pin_memory=True)
            if old is not None and rows:
                h[:rows].copy_(old[k][:rows])
            out.append(h)
    return out


def _samples_to_host(run_chunk, cuts, dev):
    """run_chunk(a, b) -> the device samples of rays [a, b), enqueued on the
    current stream; every chunk's samples are copied to pinned host memory on
    a copy stream while the next chunk runs.  Returns the numpy 9-tuple of
    the whole frame (offsets rebased, samples in ray order)."""
    m = cuts[-1]
    main = torch.cuda.current_stream()
    cp = _copy_stream(dev)
    host, cap, R0, keep, bases = None, 0, 0, [], []
    for a, b in zip(cuts[:-1], cuts[1:]):
        s = run_chunk(a, b)
        Rc = int(s[1].shape[0])
        if host is None or R0 + Rc > cap:  # first chunk (or a short guess): size from the density so far
            guess = int((R0 + Rc) * m / max(b, 1) * E2E_HEADROOM) + 1024
            cap = max(guess, int(_R_PER_RAY.get(dev, 0.0) * m * 1.05) + 1024, R0 + Rc)
            cp.synchronize()
            host = _host_buffers(s, m, cap, host, R0)
        cp.wait_event(main.record_event())
        with torch.cuda.stream(cp):
            host[0][a:b].copy_(s[0][:b - a], non_blocking=True)
            host[8][a:b].copy_(s[8], non_blocking=True)
            for k in range(1, len(s)):
                if k != 8 and s[k].shape[0] == Rc and Rc:
                    host[k][R0:R0 + Rc].copy_(s[k], non_blocking=True)
        keep.append(s)  # the device results stay alive until their copies are done
        bases.append((a, b, R0))
        R0 += Rc
    cp.synchronize()
    off = host[0].numpy()
    for a, b, base in bases:
        if base:
            off[a:b] += base
    off[m] = R0
    _R_PER_RAY[dev] = R0 / max(m, 1)
    return tuple(h.numpy() if (k in (0, 8) or h.shape[0] == 0) else h.numpy()[:R0]
                 for k, h in enumerate(host))


H2D_PIECE = int(os.environ.get("HP_H2D_PIECE", str(1 << 20)))  # bytes per staged piece of a pageable upload
_INFLIGHT: list = []  # (pinned staging block, event): blocks an upload's DMA may still read
_INFLIGHT_LOCK = threading.Lock()


def _h2d(a, dev, dtype) -> torch.Tensor:
    """Upload host data (numpy array or CPU tensor, pinned or not) to ``dev``
    on the current stream.  Pinned tensors go up directly; pageable data goes
    through hp_host_upload: host threads stage it into pinned memory piece by
    piece and each piece's DMA is enqueued as soon as it is staged (the
    driver's own pageable path runs at ~11-20 GB/s on the B200 box)."""
    if isinstance(a, torch.Tensor):
        if a.is_pinned() or a.numel() * a.element_size() < H2D_PIECE:
            return a.to(device=dev, dtype=dtype, non_blocking=True)
        a = a.numpy() if a.dtype == dtype else a.to(dtype).numpy()
    arr = np.asarray(a)
    np_dt = torch.empty((), dtype=dtype).numpy().dtype
    if arr.dtype != np_dt or not arr.flags.c_contiguous:
        arr = np.ascontiguousarray(arr, dtype=np_dt)
    if arr.nbytes < H2D_PIECE or not H2D_STAGED:
        return torch.from_numpy(arr).to(dev, non_blocking=True)  # the driver's pageable path (~20 GB/s here)
    with _INFLIGHT_LOCK:  # release the staging blocks whose copies have run
        _INFLIGHT[:] = [x for x in _INFLIGHT if not x[1].query()]
    stage = torch.empty(arr.nbytes, dtype=torch.uint8, pin_memory=True)  # caching host allocator: reused
    out = torch.empty(arr.shape, dtype=dtype, device=dev)
    stream = torch.cuda.current_stream(dev)
    lib = device._lib.load(require_device=True)
    device._lib.check(lib.hp_host_upload(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(arr.ctypes.data),
                                         arr.nbytes, ctypes.c_void_p(stage.data_ptr()), H2D_PIECE, H2D_THREADS,
                                         ctypes.c_void_p(stream.cuda_stream)))
    ev = stream.record_event()
    with _INFLIGHT_LOCK:  # torch does not see these DMAs: keep the block until they ran
        _INFLIGHT.append((stage, ev))
    return out


_COORD: list = []


def _h2d_async(stream, dev, *items):
    """:func:`_h2d` of every (host data, dtype) item on ``stream`` from a
    coordinator thread, so the host staging overlaps the caller's own work.
    Returns wait() -> the device tensors, after making the current stream
    wait for the uploads."""
    if not _COORD:
        from concurrent.futures import ThreadPoolExecutor
        _COORD.append(ThreadPoolExecutor(max_workers=1, thread_name_prefix="hp-upload"))

    def run():
        with torch.cuda.device(dev), torch.cuda.stream(stream):
            outs = [None if a is None else _h2d(a, dev, dt) for a, dt in items]
            return outs, stream.record_event()
    fut = _COORD[0].submit(run)

    def wait():
        outs, ev = fut.result()
        torch.cuda.current_stream().wait_event(ev)
        return outs
    return wait


def _host_rays(a, m, dtype, cols=None):
    """CPU torch tensor view of a per-ray host input (numpy / tensor / scalar)."""
    if isinstance(a, torch.Tensor) and a.numel() == m * (cols or 1):
        t = a.reshape(m, cols) if cols else a.reshape(m)
        return t if t.dtype == dtype else t.to(dtype)
    arr = a.numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    if arr.ndim == 0 and not cols:
        arr = np.broadcast_to(arr.astype(np.float64), (m,))
    t = torch.from_numpy(np.ascontiguousarray(arr)).reshape((m, cols) if cols else (m,))
    return t if t.dtype == dtype else t.to(dtype)


def search_and_sample(cloud, camera, search_cfg, pixels, dirs, t_near, t_far,
                      sampler_cfg: SamplerConfig | None = None, with_colors: bool = True,
                      exact_t_end: bool = True, max_matches: int | None = None):
    """Host arrays in, host arrays out: build the index for ``camera``, query
    the rays and run primary-surface sampling.  Returns the numpy 9-tuple of
    ``sample_batch_arrays`` (reference sampler.py:196-217).

    Inputs may be numpy arrays or (preferably pinned) CPU torch tensors.  The
    device build and the ray uploads are enqueued first (pageable inputs are
    staged through pinned memory by host threads, :func:`_h2d`); each chunk's
    slopes are computed on the device from its uploaded pixels
    (hp_radius_slopes, bit-identical to the reference's ``radius_slopes``).
    The frame runs in ray chunks whose result copies (pinned buffers) overlap
    the next chunk's device work (``E2E_CUTS``).
    """
    dev = torch.device("cuda", torch.cuda.current_device())
    main = torch.cuda.current_stream()
    side = _side_stream(dev)  # persistent: the caching allocator pools blocks per stream
    side.wait_stream(main)
    xyz = _h2d(cloud.positions, dev, torch.float64)          # the critical path: the build needs it
    idx = device.build_layout(xyz, camera, search_cfg.pad)   # async on the stream
    px_host = pixels.numpy() if isinstance(pixels, torch.Tensor) else np.asarray(pixels)
    px_host = np.ascontiguousarray(px_host, dtype=np.int64).reshape(-1, 2)
    m = px_host.shape[0]
    cuts = _ray_chunks(m)
    # uploads on a coordinator thread, in the order the device needs them: the
    # first chunk's rays (while the build runs and the host slopes are
    # computed), the colours (the first chunk's sampler), the other chunks' rays
    h_rays = (_host_rays(pixels, m, torch.int64, 2), _host_rays(dirs, m, torch.float64, 3),
              _host_rays(t_near, m, torch.float64), _host_rays(t_far, m, torch.float64))
    kinds = (torch.int64, torch.float64, torch.float64, torch.float64)
    ray_up = [_h2d_async(side, dev, *[(h[cuts[0]:cuts[1]], k) for h, k in zip(h_rays, kinds)])]
    cols_up = _h2d_async(side, dev, (cloud.colors if with_colors else None, torch.float64))
    ray_up += [_h2d_async(side, dev, *[(h[a:b], k) for h, k in zip(h_rays, kinds)])
               for a, b in zip(cuts[1:-1], cuts[2:])]
    cfg = sampler_cfg or SamplerConfig()
    col = []
    chunk_of = {a: i for i, a in enumerate(cuts[:-1])}

    def colours():  # resolved by _query_sample right before its sampler
        if not col:
            col.append(cols_up()[0])
        return col[0]

    def run_chunk(a, b):
        pix_d, dirs_d, tn, tf = ray_up[chunk_of[a]]()  # waits for this chunk's uploads only
        sl = device.radius_slopes(camera, search_cfg.kernel_radius, search_cfg.use_approx_radius, pixels=pix_d)
        return _query_sample(idx, colours, pix_d, dirs_d, tn, tf, sl, cfg, exact_t_end, max_matches).samples

    return _samples_to_host(run_chunk, cuts, dev)


def search_and_sample_view(cloud, camera, search_cfg, t_near: float, t_far: float,
                           sampler_cfg: SamplerConfig | None = None, with_colors: bool = True,
                           exact_t_end: bool = True, max_matches: int | None = None):
    """A whole view: the camera's ray grid (``ray_grid(camera)``, every pixel,
    row-major, scalar t_near / t_far -- the reference CLI's
    ``generate_rays`` + renderer ``_prepare``, cli.py:127-162,
    renderer.py:113-125) and its slopes generated on the device (hp_ray_grid,
    hp_radius_slopes, bit-identical to numpy), then build -> query -> sample
    as :func:`search_and_sample`
    (ray chunks, copies overlapped).  Only the cloud (and its colours) go up;
    returns the numpy 9-tuple of ``sample_batch_arrays``."""
    dev = torch.device("cuda", torch.cuda.current_device())
    main = torch.cuda.current_stream()
    side = _side_stream(dev)
    side.wait_stream(main)
    xyz = _h2d(cloud.positions, dev, torch.float64)
    idx = device.build_layout(xyz, camera, search_cfg.pad)
    dirs, pixels, tn, tf = device.ray_grid(camera, dev, t_near=t_near, t_far=t_far)
    m = int(dirs.shape[0])
    cuts = _ray_chunks(m)
    cols_up = _h2d_async(side, dev, (cloud.colors if with_colors else None, torch.float64))
    sl = device.radius_slopes(camera, search_cfg.kernel_radius, search_cfg.use_approx_radius, dev=dev)
    cfg = sampler_cfg or SamplerConfig()
    col = []

    def colours():  # resolved by _query_sample right before its sampler
        if not col:
            col.append(cols_up()[0])
        return col[0]

    def run_chunk(a, b):
        return _query_sample(idx, colours, pixels[a:b], dirs[a:b], tn[a:b], tf[a:b], sl[a:b], cfg, exact_t_end,
                             max_matches).samples

    return _samples_to_host(run_chunk, cuts, dev)


def _views_of(n_views: int, dist=None) -> list:
    """The views this rank runs: views[rank::world] (views are independent:
    no collective on the data path)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(range(n_views))
    return list(range(n_views))[dist.get_rank()::dist.get_world_size()]


def search_and_sample_views(cloud, cameras, search_cfg, t_near: float, t_far: float,
                            sampler_cfg: SamplerConfig | None = None, with_colors: bool = True,
                            exact_t_end: bool = True, max_matches: int | None = None, dist=None):
    """A batch of views of one cloud (the reference renders one index per
    view, renderer.py:113-125 / cli.py:127-162, one view after the other):
    every view's whole ray grid, build -> query -> sample, host arrays out.

    ``search_cfg`` is one SearchConfig or one per camera.  The cloud and its
    colours go up once and stay resident; each view's index, rays and slopes
    are generated on the device.  View k's samples are copied to pinned host
    memory on a copy stream while view k + 1 runs.
    With ``dist`` (torch.distributed, one process per GPU) each rank runs
    views[rank::world].  Returns {view index: numpy 9-tuple of
    ``sample_batch_arrays``} for this rank's views."""
    dev = torch.device("cuda", torch.cuda.current_device())
    cfgs = list(search_cfg) if isinstance(search_cfg, (list, tuple)) else [search_cfg] * len(cameras)
    if len(cfgs) != len(cameras):
        raise ValueError("one search config per camera (or a single one for all)")
    mine = _views_of(len(cameras), dist)
    if not mine:
        return {}
    main = torch.cuda.current_stream()
    side = _side_stream(dev)
    side.wait_stream(main)
    xyz = _h2d(cloud.positions, dev, torch.float64)
    cols_up = _h2d_async(side, dev, (cloud.colors if with_colors else None, torch.float64))
    cfg_s = sampler_cfg or SamplerConfig()
    cp = _copy_stream(dev)
    col, out, pending = [], {}, []

    def colours():
        if not col:
            col.append(cols_up()[0])
        return col[0]

    for i in mine:
        cam, cfg = cameras[i], cfgs[i]
        idx = device.build_layout(xyz, cam, cfg.pad)
        dirs, pixels, tn, tf = device.ray_grid(cam, dev, t_near=t_near, t_far=t_far)
        sl = device.radius_slopes(cam, cfg.kernel_radius, cfg.use_approx_radius, dev=dev)
        s = _query_sample(idx, colours, pixels, dirs, tn, tf, sl, cfg_s, exact_t_end, max_matches).samples
        R = int(s[1].shape[0])
        host = [torch.empty(tuple(x.shape), dtype=x.dtype, pin_memory=True)
                if (x.shape[0] == R and R) or k in (0, 8) else torch.zeros(tuple(x.shape), dtype=x.dtype)
                for k, x in enumerate(s)]
        cp.wait_event(main.record_event())
        with torch.cuda.stream(cp):
            for k, x in enumerate(s):
                if host[k].is_pinned():
                    host[k].copy_(x, non_blocking=True)
            done = cp.record_event()
        pending.append((i, host, s, done))  # the device results live until copied
        while pending and pending[0][3].query():
            j, h, *_ = pending.pop(0)
            out[j] = tuple(x.numpy() for x in h)
    for j, h, _, done in pending:
        done.synchronize()
        out[j] = tuple(x.numpy() for x in h)
    return out
