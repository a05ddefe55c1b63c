"""Drop-in for the reference's ``hashpoint.renderer`` (renderer.py:1-223): colour
and depth synthesis from the retained surface samples.

``render`` / ``render_volume`` / ``render_knp`` keep the reference's
signatures and results: the rays are queried and sampled on the device (the
frame path: no query CSR, retention decided with the exact early exit -- the
retained samples are the reference's bit for bit) and composited by
``hp_render`` (one thread per ray), then the image comes back to the host.
``volume_sample_weights`` is the reference's single-ray helper, kept as a
host utility for API compatibility; ``write_ppm`` / ``write_pgm16`` are the
reference's image dumps.

Values pass through log1p / exp / divisions whose last bits may differ from
glibc / numpy (compare at 1e-12 relative).  knp ties: when the k-th smallest
distance of a ray is tied, the reference's ``np.argpartition`` picks the
tied samples in an implementation-defined order; the device takes them in
sample order.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import device, pipeline
from .geometry import SearchConfig, radius_slopes
from .hash_index import HashIndex, _check_config, _check_rays, _pack_rays
from .sampler import SamplerConfig

__all__ = ["RenderConfig", "Image", "render", "render_knp", "render_volume", "volume_sample_weights",
           "write_ppm", "write_pgm16"]

MODES = ("knp_blend", "volume")


@dataclass(frozen=True)
class RenderConfig:
    """Rendering mode, background colour, and K for nearest-point blending
    (reference renderer.py:36-54)."""

    mode: str = "volume"
    background: tuple = (0.0, 0.0, 0.0)
    knp_k: int = 8

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        if self.knp_k < 1:
            raise ValueError("knp_k must be at least 1")
        bg = tuple(float(c) for c in self.background)
        if len(bg) != 3 or any(not (0.0 <= c <= 1.0) for c in bg):
            raise ValueError("background must be three channels in [0, 1]")
        object.__setattr__(self, "background", bg)


@dataclass
class Image:
    """RGB buffer in [0, 1] plus an expected-depth buffer, camera sized."""

    color: np.ndarray
    depth: np.ndarray | None
    t_near: float
    t_far: float

    @property
    def width(self) -> int:
        return self.color.shape[1]

    @property
    def height(self) -> int:
        return self.color.shape[0]


def volume_sample_weights(alphas: np.ndarray, ts: np.ndarray, t_far: float):
    """Compositing weights of one ray's samples via per-sample densities and
    the final transmittance (host helper; reference renderer.py:72-110)."""
    alphas = np.asarray(alphas, dtype=np.float64)
    ts = np.asarray(ts, dtype=np.float64)
    n = alphas.shape[0]
    weights = np.zeros(n)
    trans = 1.0
    if n == 0:
        return weights, trans
    if n == 1:
        deltas = np.array([t_far - ts[0]])
    else:
        deltas = np.append(np.diff(ts), ts[-1] - ts[-2])
    for j in range(n):
        a, dt = float(alphas[j]), float(deltas[j])
        if a >= 1.0:  # opaque: the ray ends here
            absorbed, passed = 1.0, 0.0
        elif dt > 0.0:
            passed = math.exp(-(-math.log1p(-a) / dt) * dt)
            absorbed = 1.0 - passed
        else:
            absorbed, passed = a, 1.0 - a
        weights[j] = trans * absorbed
        trans *= passed
    return weights, trans


def _render(index: HashIndex, rays: list, search_cfg, sampler_cfg, render_cfg: RenderConfig) -> Image:
    if not index.points.has_colors:
        raise ValueError("rendering requires a point cloud with colors")
    search_cfg = _check_config(index, search_cfg) if search_cfg is not None else index.config
    sampler_cfg = sampler_cfg or SamplerConfig()
    cam = index.camera
    pixels, dirs, t_near, t_far = _pack_rays(rays)
    _check_rays(index, pixels, cam.origin)  # array-level check, as query_batch_arrays
    m = pixels.shape[0]
    color = np.empty((cam.height, cam.width, 3))
    color[:, :] = render_cfg.background
    depth = np.full((cam.height, cam.width), float(t_far[0]) if m else 2.0)
    image = Image(color=color, depth=depth, t_near=float(t_near[0]) if m else 1.0,
                  t_far=float(t_far[0]) if m else 2.0)
    if m == 0:
        return image
    lib = device._lib.load(require_device=True)
    dev = index.device.device
    up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa: E731
    slopes = radius_slopes(cam, pixels, search_cfg.kernel_radius, search_cfg.use_approx_radius)
    pix_d, tf_d = up(pixels, np.int64), up(t_far, np.float64)
    pcol = up(index.points.colors, np.float64)
    # retained samples on the device (retention is decided by the exact early
    # exit: the retained set is the reference's; t_end is not needed here)
    fr = pipeline._query_sample(index.device, pcol, pix_d, up(dirs, np.float64), up(t_near, np.float64), tf_d,
                                up(slopes, np.float64), sampler_cfg, False, None)
    r_off, r_id, r_t, r_dist, _, r_alpha, _, r_color, _ = fr.samples
    col_d = up(color, np.float64)
    dep_d = up(depth, np.float64)
    owner = torch.empty(cam.width * cam.height, dtype=torch.int32, device=dev)
    bg = (ctypes.c_double * 3)(*render_cfg.background)
    p = device._ptr
    device._lib.check(lib.hp_render(1 if render_cfg.mode == "knp_blend" else 0, p(r_off), m, p(r_id), p(r_t),
                                    p(r_dist), p(r_alpha), p(r_color), p(pcol), p(pix_d), 2, p(tf_d),
                                    int(render_cfg.knp_k), bg, cam.width, cam.height, p(owner), p(col_d),
                                    p(dep_d), device._stream()))
    image.color = col_d.cpu().numpy()
    image.depth = dep_d.cpu().numpy()
    return image


def render_knp(index: HashIndex, rays: list, search_cfg: SearchConfig | None = None,
               sampler_cfg: SamplerConfig | None = None, render_cfg: RenderConfig | None = None) -> Image:
    """Blend each ray's K nearest retained points by inverse distance
    (reference renderer.py:138-160)."""
    return _render(index, rays, search_cfg, sampler_cfg, render_cfg or RenderConfig(mode="knp_blend"))


def render_volume(index: HashIndex, rays: list, search_cfg: SearchConfig | None = None,
                  sampler_cfg: SamplerConfig | None = None, render_cfg: RenderConfig | None = None) -> Image:
    """Composite retained samples front to back with density-derived weights
    (reference renderer.py:163-185)."""
    return _render(index, rays, search_cfg, sampler_cfg, render_cfg or RenderConfig(mode="volume"))


def render(index: HashIndex, rays: list, search_cfg: SearchConfig | None = None,
           sampler_cfg: SamplerConfig | None = None, render_cfg: RenderConfig | None = None) -> Image:
    """Dispatch on ``render_cfg.mode`` (reference renderer.py:188-202)."""
    render_cfg = render_cfg or RenderConfig()
    if render_cfg.mode == "knp_blend":
        return render_knp(index, rays, search_cfg, sampler_cfg, render_cfg)
    return render_volume(index, rays, search_cfg, sampler_cfg, render_cfg)


def write_ppm(image: Image, path) -> None:
    """Binary PPM (P6, 8-bit) colour dump."""
    data = np.rint(np.clip(image.color, 0.0, 1.0) * 255.0).astype(np.uint8)
    with open(path, "wb") as fh:
        fh.write(f"P6\n{image.width} {image.height}\n255\n".encode("ascii"))
        fh.write(data.tobytes())


def write_pgm16(image: Image, path) -> None:
    """Binary PGM (P5, 16-bit big-endian) depth dump over [t_near, t_far]."""
    if image.depth is None:
        raise ValueError("image has no depth buffer")
    norm = np.clip((image.depth - image.t_near) / (image.t_far - image.t_near), 0.0, 1.0)
    data = np.rint(norm * 65535.0).astype(">u2")
    with open(path, "wb") as fh:
        fh.write(f"P5\n{image.width} {image.height}\n65535\n".encode("ascii"))
        fh.write(data.tobytes())
