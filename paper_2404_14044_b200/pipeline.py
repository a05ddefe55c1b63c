"""Chained search -> sampling, the way the reference's renderer drives the path
(renderer._prepare, reference renderer.py:113-125: query_batch_arrays then
sample_batch_arrays on the same CSR).

Here the query CSR never leaves HBM: only rays/points go up and the retained
samples come back.  ``frame_device`` is the all-device step the benchmark
times; ``search_and_sample`` is the host-buffer public entry point (numpy in,
numpy out) used for the end-to-end number.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device
from .geometry import radius_slopes
from .sampler import SamplerConfig

__all__ = ["FrameResult", "frame_device", "search_and_sample", "StageTimer"]


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
    query: tuple
    samples: tuple

    @property
    def Q(self) -> int:
        return int(self.query[1].numel())

    @property
    def R(self) -> int:
        return int(self.samples[1].numel())


def frame_device(xyz: torch.Tensor, colors: torch.Tensor | None, camera, search_cfg, pixels,
                 dirs, t_near, t_far, slopes, sampler_cfg: SamplerConfig | None = None,
                 exact_t_end: bool = True, timer: StageTimer | None = None) -> FrameResult:
    """build -> query -> sample, all on the device (CUDA tensors in and out)."""
    sampler_cfg = sampler_cfg or SamplerConfig()
    mark = timer.mark if timer is not None else (lambda name: None)
    mark("start")
    idx = device.build(xyz, camera, search_cfg.pad)
    mark("build")
    q = device.query(idx, pixels, dirs, t_near, t_far, slopes)
    mark("query")
    s = device.sample(q[0], q[1], q[2], q[3], slopes, sampler_cfg, colors, exact_t_end)
    mark("sample")
    return FrameResult(idx, q, s)


def search_and_sample(cloud, camera, search_cfg, pixels, dirs, t_near, t_far,
                      sampler_cfg: SamplerConfig | None = None, with_colors: bool = True,
                      exact_t_end: bool = True):
    """Host arrays in, host arrays out: build the index for ``camera``, query
    the rays and run primary-surface sampling.  Returns the numpy 9-tuple of
    ``sample_batch_arrays`` (reference sampler.py:196-217)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    pixels = np.ascontiguousarray(pixels, dtype=np.int64).reshape(-1, 2)
    m = pixels.shape[0]
    slopes = radius_slopes(camera, pixels, search_cfg.kernel_radius, search_cfg.use_approx_radius)

    def up(a, dt, shape=None):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=dt))
        return t.to(dev, non_blocking=True) if shape is None else t.to(dev).view(*shape)

    xyz = up(cloud.positions, np.float64)
    col = up(cloud.colors, np.float64) if (with_colors and cloud.colors is not None) else None
    fr = frame_device(xyz, col, camera, search_cfg, up(pixels, np.int64), up(dirs, np.float64),
                      up(np.broadcast_to(t_near, (m,)), np.float64),
                      up(np.broadcast_to(t_far, (m,)), np.float64), up(slopes, np.float64),
                      sampler_cfg, exact_t_end)
    return tuple(x.cpu().numpy() for x in fr.samples)
