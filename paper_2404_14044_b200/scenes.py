"""Seeded synthetic point clouds and the look-at camera used by the benchmarks.

The generators reproduce the reference's recipes draw-for-draw
(``scenes.py:63-98``: one ``np.random.default_rng(seed)`` stream, identical call
order and expression order), so a ``SceneSpec`` yields the same float64 cloud
in both packages and the golden fixtures stay meaningful.  ``ply_file`` scenes
(file IO) are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .cloud import PointCloud
from .geometry import Camera

__all__ = ["SceneSpec", "generate_scene", "scene_camera", "PLANE_PALETTE"]

PLANE_PALETTE = np.array([(0.9, 0.2, 0.2), (0.2, 0.9, 0.2), (0.2, 0.2, 0.9),
                          (0.8, 0.8, 0.2), (0.8, 0.2, 0.8), (0.2, 0.8, 0.8)])

_KINDS = ("uniform_box", "sphere_surface", "parallel_planes")


@dataclass(frozen=True)
class SceneSpec:
    kind: str
    n: int = 1000
    seed: int = 0
    noise: float = 0.0
    center: tuple = (0.0, 0.0, 4.0)
    extent: float = 2.0
    sphere_radius: float = 1.0
    plane_count: int = 2
    plane_gap: float = 0.5

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ValueError(f"kind must be one of {_KINDS}")
        if self.n < 0 or self.noise < 0 or self.extent <= 0:
            raise ValueError("need n >= 0, noise >= 0, extent > 0")
        if self.kind == "parallel_planes" and self.plane_count < 1:
            raise ValueError("plane_count must be at least 1")


def _jitter(rng, sigma, count):
    # surface noise, clipped at 4 sigma; no draw at all when sigma == 0
    if sigma == 0.0:
        return np.zeros(count)
    return np.clip(rng.normal(0.0, sigma, count), -4.0 * sigma, 4.0 * sigma)


def _box(spec, rng, c):
    h = 0.5 * spec.extent
    xyz = c + rng.uniform(-h, h, (spec.n, 3))
    return xyz, rng.uniform(0.0, 1.0, (spec.n, 3))


def _sphere(spec, rng, c):
    unit = rng.normal(size=(spec.n, 3))
    lens = np.linalg.norm(unit, axis=1, keepdims=True)
    lens[lens == 0] = 1.0
    unit /= lens
    rad = spec.sphere_radius + _jitter(rng, spec.noise, spec.n)
    return c + unit * rad[:, None], 0.5 + 0.5 * unit


def _planes(spec, rng, c):
    k = spec.plane_count
    first_z = c[2] - 0.5 * (k - 1) * spec.plane_gap
    sizes = np.full(k, spec.n // k)
    sizes[: spec.n % k] += 1
    h = 0.5 * spec.extent
    xyz, rgb = [], []
    for i, cnt in enumerate(int(s) for s in sizes):
        xy = c[:2] + rng.uniform(-h, h, (cnt, 2))
        z = first_z + i * spec.plane_gap + _jitter(rng, spec.noise, cnt)
        xyz.append(np.column_stack([xy, z]))
        rgb.append(np.tile(PLANE_PALETTE[i % len(PLANE_PALETTE)], (cnt, 1)))
    if not xyz:
        return np.zeros((0, 3)), np.zeros((0, 3))
    return np.concatenate(xyz), np.concatenate(rgb)


_GENERATORS = {"uniform_box": _box, "sphere_surface": _sphere, "parallel_planes": _planes}


def generate_scene(spec: SceneSpec) -> PointCloud:
    rng = np.random.default_rng(spec.seed)
    xyz, rgb = _GENERATORS[spec.kind](spec, rng, np.asarray(spec.center, dtype=np.float64))
    return PointCloud(xyz, rgb)


def scene_camera(width: int = 64, height: int = 64, fov_deg: float = 40.0,
                 origin=(0.0, 0.0, 0.0), target=(0.0, 0.0, 4.0),
                 up=(0.0, 1.0, 0.0), focal_length: float = 1.0) -> Camera:
    """Square-pixel look-at camera; ``fov_deg`` spans the image width."""
    o = np.asarray(origin, dtype=np.float64)
    pix = 2.0 * focal_length * np.tan(np.radians(fov_deg) / 2.0) / width
    return Camera.from_vectors(o, np.asarray(target, dtype=np.float64) - o, up,
                               focal_length, width, height, pix, pix)
