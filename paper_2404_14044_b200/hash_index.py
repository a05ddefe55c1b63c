"""Drop-in for the reference's ``hashpoint.hash_index`` (hash_index.py:1-304).

Same entry points, argument meaning, dtypes, result layout and ValueError
messages; the work runs on the B200 through libhp_b200.so:

  build               hash_index.py:151-190   -> device.build (hp_build)
  query_batch_arrays  hash_index.py:212-235   -> device.query (hp_query_count/fill)
  query               hash_index.py:252-260
  query_batch         hash_index.py:263-293   (one device batch; ``parallel`` is
                                               accepted and has no effect on results)

``HashIndex`` keeps its arrays in HBM and materialises the reference's numpy
fields (table_start, ..., slot_z) on first access.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, device
from .cloud import PointCloud
from .geometry import Camera, Ray, SearchConfig, radius_slopes

__all__ = ["QueryResult", "HashIndex", "build", "query", "query_batch", "query_batch_arrays",
           "results_from_csr", "morton_codes", "rasterize_points"]


def _frozen(a: np.ndarray) -> np.ndarray:
    a.flags.writeable = False
    return a


@dataclass(frozen=True)
class QueryResult:
    """Neighbours of one ray, sorted by t_proj (ties by id); ids unique."""

    point_ids: np.ndarray
    t_proj: np.ndarray
    dist_perp: np.ndarray

    def __post_init__(self):
        ids = np.ascontiguousarray(self.point_ids, dtype=np.int64)
        t = np.ascontiguousarray(self.t_proj, dtype=np.float64)
        d = np.ascontiguousarray(self.dist_perp, dtype=np.float64)
        if ids.ndim != 1 or not (ids.shape == t.shape == d.shape):
            raise ValueError("point_ids, t_proj, dist_perp must be equal-length 1-D arrays")
        object.__setattr__(self, "point_ids", _frozen(ids))
        object.__setattr__(self, "t_proj", _frozen(t))
        object.__setattr__(self, "dist_perp", _frozen(d))

    def __len__(self) -> int:
        return int(self.point_ids.shape[0])

    @classmethod
    def empty(cls) -> "QueryResult":
        return cls(np.empty(0, np.int64), np.empty(0), np.empty(0))


def results_from_csr(offsets, ids, t, dist) -> list:
    offsets = np.asarray(offsets)
    return [QueryResult(ids[a:b], t[a:b], dist[a:b])
            for a, b in zip(offsets[:-1].tolist(), offsets[1:].tolist())]


def _spread_bits(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64) & np.uint64(0xFFFF)
    for shift, mask in ((8, 0x00FF00FF), (4, 0x0F0F0F0F), (2, 0x33333333), (1, 0x55555555)):
        x = (x | (x << np.uint64(shift))) & np.uint64(mask)
    return x


def morton_codes(u: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Z-order code of 16-bit (u, v): u bits even, v bits odd (host utility)."""
    return (_spread_bits(u) | (_spread_bits(v) << np.uint64(1))).astype(np.int64)


def rasterize_points(positions: np.ndarray, camera: Camera, pad: int):
    """Host (numpy) rasterization, for tests/inspection only; the device build
    evaluates the same expressions in a fixed order."""
    wp, hp = camera.width + 2 * pad, camera.height + 2 * pad
    u, v, depth = camera.project(positions)
    fu, fv = np.floor(u) + pad, np.floor(v) + pad
    ok = (depth > 0) & (fu >= 0) & (fu < wp) & (fv >= 0) & (fv < hp)
    return ok, np.where(ok, fu, 0).astype(np.int64), np.where(ok, fv, 0).astype(np.int64)


_FIELDS = ("table_start", "table_count", "reordered_ids", "slot_x", "slot_y", "slot_z")


class HashIndex:
    """Immutable search index (reference hash_index.py:115-148).

    ``device`` holds the HBM-resident arrays; the numpy fields of the
    reference are copied to the host lazily, once.
    """

    __slots__ = ("points", "camera", "config", "pad", "_touch_n", "device", "_host")

    def __init__(self, points, camera, config, dev: device.DeviceIndex):
        object.__setattr__(self, "points", points)
        object.__setattr__(self, "camera", camera)
        object.__setattr__(self, "config", config)
        object.__setattr__(self, "pad", int(dev.pad))
        object.__setattr__(self, "_touch_n", int(points.count))
        object.__setattr__(self, "device", dev)
        object.__setattr__(self, "_host", {})

    def __setattr__(self, name, value):
        raise AttributeError("HashIndex is immutable")

    def __getattr__(self, name):
        if name in _FIELDS:
            host = object.__getattribute__(self, "_host")
            if name not in host:
                host[name] = _frozen(getattr(object.__getattribute__(self, "device"), name)
                                     .cpu().numpy())
            return host[name]
        raise AttributeError(name)

    @property
    def point_touches(self) -> int:
        """Per-point visits of the three build passes: n + 2 N_in (hash_index.py:189)."""
        return self._touch_n + 2 * int(self.device.n_in)

    @property
    def padded_width(self) -> int:
        return self.camera.width + 2 * self.pad

    @property
    def padded_height(self) -> int:
        return self.camera.height + 2 * self.pad

    @property
    def indexed_count(self) -> int:
        return int(self.device.n_in)


def _device():
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None


def build(points: PointCloud, camera: Camera, config: SearchConfig) -> HashIndex:
    """Rasterize ``points`` for ``camera`` and build the lookup table on the GPU."""
    pad = config.pad
    if max(camera.width + 2 * pad, camera.height + 2 * pad) > 0xFFFF:
        raise ValueError("padded image exceeds 16-bit pixel coordinates")
    _lib.load(require_device=True)
    pos = np.ascontiguousarray(points.positions, dtype=np.float64)
    if not pos.flags.writeable:  # frozen cloud arrays: torch wants a writable buffer to wrap
        pos = pos.copy()
    dev = device.build(torch.from_numpy(pos).to(_device(), non_blocking=False), camera, pad)
    return HashIndex(points, camera, config, dev)


def _check_config(index: HashIndex, config):
    if config is None:
        return index.config
    if config.kernel_size != index.config.kernel_size:
        raise ValueError(f"config kernel size {config.kernel_size} does not match the "
                         f"index padding (built with {index.config.kernel_size})")
    return config


def _check_rays(index: HashIndex, pixels: np.ndarray, origin) -> None:
    cam = index.camera
    if not np.array_equal(origin, cam.origin):
        raise ValueError("ray origin differs from the index camera origin")
    if pixels.size and (pixels[:, 0].min() < 0 or pixels[:, 0].max() >= cam.width
                        or pixels[:, 1].min() < 0 or pixels[:, 1].max() >= cam.height):
        raise ValueError("ray pixel outside the index camera image")


def query_batch_arrays(index: HashIndex, pixels, dirs, t_near, t_far, config=None):
    """Array-level batch query; returns numpy
    ``(offsets, ids, t_proj, dist_perp, probes, scanned)`` (hash_index.py:212-235)."""
    config = _check_config(index, config)
    pixels = np.ascontiguousarray(pixels, dtype=np.int64).reshape(-1, 2)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    _check_rays(index, pixels, index.camera.origin)
    slopes = radius_slopes(index.camera, pixels, config.kernel_radius, config.use_approx_radius)
    out = query_device_arrays(index, pixels, dirs, t_near, t_far, slopes)
    return tuple(o.cpu().numpy() for o in out)


def query_device_arrays(index: HashIndex, pixels, dirs, t_near, t_far, slopes):
    """Host arrays in, CUDA tensors out (H2D of the rays, no D2H)."""
    dev = index.device.device

    def up(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        if not a.flags.writeable:  # broadcast / frozen views: torch wants a writable buffer
            a = a.copy()
        return torch.from_numpy(a).to(dev)

    m = int(np.asarray(pixels).shape[0])
    return device.query(index.device, up(pixels, np.int64).view(m, 2), up(dirs, np.float64).view(m, 3),
                        up(np.broadcast_to(t_near, (m,)), np.float64),
                        up(np.broadcast_to(t_far, (m,)), np.float64), up(slopes, np.float64))


def _pack_rays(rays: list):
    m = len(rays)
    pixels = np.empty((m, 2), np.int64)
    dirs = np.empty((m, 3), np.float64)
    t_near = np.empty(m)
    t_far = np.empty(m)
    for i, r in enumerate(rays):
        pixels[i] = r.pixel
        dirs[i] = r.direction
        t_near[i] = r.t_near
        t_far[i] = r.t_far
    return pixels, dirs, t_near, t_far


def query(index: HashIndex, ray: Ray, config=None) -> QueryResult:
    if not np.array_equal(ray.origin, index.camera.origin):
        raise ValueError("ray origin differs from the index camera origin")
    offsets, ids, t, dist, _, _ = query_batch_arrays(index, *_pack_rays([ray]), config)
    return QueryResult(ids, t, dist)


def query_batch(index: HashIndex, rays: list, config=None, parallel: bool = False) -> list:
    """Element-wise :func:`query` in input order.  The GPU processes the whole
    batch at once; ``parallel`` (thread chunking in the reference) is accepted
    for API compatibility and does not change results."""
    for r in rays:
        if not np.array_equal(r.origin, index.camera.origin):
            raise ValueError("ray origin differs from the index camera origin")
    offsets, ids, t, dist, _, _ = query_batch_arrays(index, *_pack_rays(rays), config)
    return results_from_csr(offsets, ids, t, dist)
