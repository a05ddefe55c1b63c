"""Drop-in for the reference's ``hashpoint.sampler`` (sampler.py:1-226).

``sample_batch_arrays`` (sampler.py:196-217) and ``sample_ray``
(sampler.py:182-193) run on the B200 (hp_sample_run/emit).  The scalar stage
functions (``make_candidates``, ``pseudo_udf``, ``confidence``,
``occlusion_weights``, ``retain``) are the reference's readable single-ray
restatement (sampler.py:90-179); they are host utilities kept for API
compatibility, not part of the accelerated path.

``sample_batch_arrays(..., exact_t_end=True)`` reproduces the reference's
``transmittance`` over all candidates.  With ``exact_t_end=False`` each ray
stops once retention is decided; every retained output is unchanged and the
returned transmittance is the value at that point.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import device
from .geometry import Camera, Ray, SearchConfig, radius_slope, radius_slopes
from .hash_index import HashIndex, QueryResult, query_device_arrays, _pack_rays, _check_config

__all__ = ["SamplerConfig", "SampleCandidate", "make_candidates", "pseudo_udf", "confidence",
           "occlusion_weights", "retain", "sample_ray", "sample_batch_arrays",
           "primary_surface"]

DEFAULT_BETA_SQ = 0.02


@dataclass(frozen=True)
class SamplerConfig:
    """Sampling hyper-parameters (reference sampler.py:37-68)."""

    k_neighbors: int = 8
    beta: float = math.sqrt(DEFAULT_BETA_SQ)
    gamma: float = 0.9
    retention_mode: str = "epsilon"
    epsilon: float = 1e-4
    tau_min: float = 0.01

    def __post_init__(self):
        if self.k_neighbors < 1:
            raise ValueError("k_neighbors must be at least 1")
        if self.beta <= 0:
            raise ValueError("beta must be positive")
        if not 0.0 < self.gamma <= 1.0:
            raise ValueError("gamma must be in (0, 1]")
        if self.retention_mode not in ("epsilon", "tau"):
            raise ValueError("retention_mode must be 'epsilon' or 'tau'")
        if self.epsilon < 0:
            raise ValueError("epsilon must be non-negative")
        if not 0.0 <= self.tau_min < 1.0:
            raise ValueError("tau_min must be in [0, 1)")


@dataclass
class SampleCandidate:
    t: float
    position: np.ndarray
    radius: float
    dist_perp: float
    point_id: int
    udf_distance: float | None = None
    confidence: float | None = None
    weight: float | None = None


# ---------------------------------------------------------------- host helpers
def make_candidates(result: QueryResult, ray: Ray, camera: Camera, config: SearchConfig) -> list:
    slope = radius_slope(camera, ray.pixel, config.kernel_radius, config.use_approx_radius)
    cands = [SampleCandidate(t=float(t), position=ray.origin + float(t) * ray.direction,
                             radius=slope * float(t), dist_perp=float(d), point_id=int(i))
             for i, t, d in zip(result.point_ids, result.t_proj, result.dist_perp)]
    cands.sort(key=lambda c: c.t)
    return cands


def pseudo_udf(candidate: SampleCandidate, neighbors: QueryResult, k: int) -> float:
    """Mean distance from the candidate to its k nearest retrieved points
    (eligible = within the candidate's radius when at least k exist)."""
    if len(neighbors) == 0:
        raise ValueError("candidate needs at least one retrieved neighbor")
    if k < 1:
        raise ValueError("k must be at least 1")
    d2 = (neighbors.t_proj - candidate.t) ** 2 + neighbors.dist_perp ** 2
    inside = neighbors.dist_perp <= candidate.radius
    pool = d2[inside] if int(inside.sum()) >= k else d2
    kk = min(k, pool.shape[0])
    return float(np.mean(np.sqrt(np.partition(pool, kk - 1)[:kk])))


def confidence(udf_distance: float, beta: float, gamma: float) -> float:
    if beta <= 0:
        raise ValueError("beta must be positive")
    if not 0.0 < gamma <= 1.0:
        raise ValueError("gamma must be in (0, 1]")
    if udf_distance < 0:
        raise ValueError("distance must be non-negative")
    return gamma * math.exp(-(udf_distance * udf_distance) / (beta * beta))


def occlusion_weights(candidates: list) -> list:
    last = -math.inf
    for c in candidates:
        if c.confidence is None:
            raise ValueError("candidate confidences must be set first")
        if c.t < last:
            raise ValueError("candidates must be sorted by t ascending")
        last = c.t
    trans = 1.0
    for c in candidates:
        c.weight = c.confidence * trans
        trans *= 1.0 - c.confidence
    return candidates


def retain(candidates: list, config: SamplerConfig) -> list:
    if config.retention_mode == "epsilon":
        return [c for c in candidates if c.weight >= config.epsilon]
    kept, trans = [], 1.0
    for c in candidates:
        if trans < config.tau_min:
            break
        kept.append(c)
        trans *= 1.0 - c.confidence
    return kept


# ---------------------------------------------------------------- device path
_NP = {torch.int64: np.int64, torch.float64: np.float64}


def _to_dev(a, dt, dev):
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dt).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=_NP[dt])).to(dev)


def sample_batch_device(offsets, ids, t_proj, dist_perp, slopes, sampler_cfg: SamplerConfig,
                        colors=None, exact_t_end: bool = True):
    """Like :func:`sample_batch_arrays` but returns CUDA tensors."""
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
    if dev is None:
        device._lib.load(require_device=True)
    o = _to_dev(offsets, torch.int64, dev)
    col = None if colors is None else _to_dev(colors, torch.float64, dev).view(-1, 3)
    return device.sample(o, _to_dev(ids, torch.int64, dev), _to_dev(t_proj, torch.float64, dev),
                         _to_dev(dist_perp, torch.float64, dev), _to_dev(slopes, torch.float64, dev),
                         sampler_cfg, col, exact_t_end)


def sample_batch_arrays(offsets, ids, t_proj, dist_perp, slopes, sampler_cfg: SamplerConfig,
                        colors=None, *, exact_t_end: bool = True):
    """Batch sampling over CSR query results (reference sampler.py:196-217).

    Returns numpy ``(offsets, point_ids, t, dist_perp, udf, alpha, weight,
    color, transmittance)``; ``color`` is (0, 3) unless ``colors`` is given.
    """
    out = sample_batch_device(offsets, ids, t_proj, dist_perp, slopes, sampler_cfg, colors,
                              exact_t_end)
    return tuple(x.cpu().numpy() for x in out)


def sample_ray(index: HashIndex, ray: Ray, search_cfg: SearchConfig | None = None,
               sampler_cfg: SamplerConfig | None = None) -> list:
    """Query + full sampling pipeline for one ray (reference sampler.py:182-193)."""
    search_cfg = _check_config(index, search_cfg) if search_cfg is not None else index.config
    sampler_cfg = sampler_cfg or SamplerConfig()
    if not np.array_equal(ray.origin, index.camera.origin):
        raise ValueError("ray origin differs from the index camera origin")
    pixels, dirs, tn, tf = _pack_rays([ray])
    slopes = radius_slopes(index.camera, pixels, search_cfg.kernel_radius,
                           search_cfg.use_approx_radius)
    q = query_device_arrays(index, pixels, dirs, tn, tf, slopes)
    r_off, r_id, r_t, r_dist, r_udf, r_alpha, r_w, _, _ = (
        x.cpu().numpy() for x in device.sample(q[0], q[1], q[2], q[3], q[0].new_tensor(
            slopes, dtype=torch.float64), sampler_cfg))
    slope = radius_slope(index.camera, ray.pixel, search_cfg.kernel_radius,
                         search_cfg.use_approx_radius)
    return [SampleCandidate(t=float(r_t[k]), position=ray.origin + float(r_t[k]) * ray.direction,
                            radius=slope * float(r_t[k]), dist_perp=float(r_dist[k]),
                            point_id=int(r_id[k]), udf_distance=float(r_udf[k]),
                            confidence=float(r_alpha[k]), weight=float(r_w[k]))
            for k in range(len(r_id))]


def primary_surface(r_off, r_id, r_t):
    """First retained candidate per ray: numpy ``(point_id or -1, t or NaN)``."""
    r_off = np.asarray(r_off)
    r_id = np.asarray(r_id)
    r_t = np.asarray(r_t)
    has = r_off[1:] > r_off[:-1]
    first = np.minimum(r_off[:-1], max(len(r_id) - 1, 0))
    pid = np.where(has, r_id[first] if len(r_id) else -1, -1).astype(np.int64)
    pt = np.where(has, r_t[first] if len(r_t) else np.nan, np.nan)
    return pid, pt
