"""Point-NeRF-style feature aggregation on the sampler's output (cfg5, the
"full render step": search + primary-surface sampling + aggregation MLP).

The paper plugs its search and sampling into Point-NeRF, whose MLP turns the
features of each sample's neighbouring points into density and colour
(PAPER.md:256-259, :325).  The reference package stops at the sampler
(SPEC.md:15), so this module defines the aggregation concretely, after
Point-NeRF: per retained sample s with neighbours i (the sampler's K nearest,
``emit_knn``) and blend weights w_si,

    in_si = [f_i | sin/cos(2^l pi (p_i - x_s)), l < 4 | p_i - x_s | 1 | 0 x 4]   (64)
    h2_si = relu(W2 relu(W1 in_si) + b2)                                         (128)
    g_s   = sum_i w_si h2_si                                                     (128)
    (sigma, rgb) = (softplus, sigmoid)(W4 relu(W3 g_s + b3) + b4)

with bf16 operands and fp32 accumulation on the tensor cores
(``hp_pointnerf_aggregate`` / ``hp_pointnerf_head``, tcgen05 + TMEM), and
an fp32 PyTorch restatement (:meth:`PointNeRFMLP.reference`) as the parity
oracle.  Weights and point features are random (seeded): there is no
checkpoint to load.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib, device

__all__ = ["PointNeRFMLP", "sample_rays", "render_step"]

FEAT, IN, HID, HEAD = 32, 64, 128, 64


def sample_rays(r_off: torch.Tensor) -> torch.Tensor:
    """int32 [R]: the ray of every retained sample (from the CSR offsets)."""
    m = int(r_off.shape[0]) - 1
    counts = r_off[1:] - r_off[:-1]
    R = int(r_off[-1].item()) if m > 0 else 0
    return torch.repeat_interleave(torch.arange(m, dtype=torch.int32, device=r_off.device), counts,
                                   output_size=R)


class PointNeRFMLP:
    """The aggregation MLP's parameters (bf16 where the tensor cores read
    them) and the per-point features, on ``device``."""

    def __init__(self, n_points: int, seed: int = 0, device_=None):
        dev = device_ or torch.device("cuda", torch.cuda.current_device())
        g = torch.Generator().manual_seed(seed)

        def rnd(*shape, scale=1.0):
            return (torch.randn(*shape, generator=g, dtype=torch.float32) * scale)

        self.w1 = rnd(HID, IN, scale=1.0 / math.sqrt(IN)).to(torch.bfloat16).to(dev)
        self.w2 = rnd(HID, HID, scale=1.0 / math.sqrt(HID)).to(torch.bfloat16).to(dev)
        self.b2 = rnd(HID, scale=0.1).to(dev)
        self.w3 = rnd(HEAD, HID, scale=1.0 / math.sqrt(HID)).to(torch.bfloat16).to(dev)
        self.b3 = rnd(HEAD, scale=0.1).to(dev)
        self.w4 = rnd(4, HEAD, scale=1.0 / math.sqrt(HEAD)).to(dev)
        self.b4 = rnd(4, scale=0.1).to(dev)
        self.features = rnd(n_points, FEAT).to(torch.bfloat16).to(dev)

    # ------------------------------------------------------------ device path
    def aggregate(self, knn_id, knn_w, sample_ray, r_t, dirs, origin, positions) -> torch.Tensor:
        """g: bf16 [R, 128] (hp_pointnerf_aggregate)."""
        lib = _lib.load(require_device=True)
        R, K = int(knn_id.shape[0]), int(knn_id.shape[1]) if knn_id.dim() == 2 else 1
        g = torch.empty((max(R, 1), HID), dtype=torch.bfloat16, device=knn_id.device)[:R]
        o = (ctypes.c_double * 3)(*[float(v) for v in np.asarray(origin, np.float64)])
        args = (knn_id.contiguous(), knn_w.contiguous(), sample_ray.contiguous(), r_t.contiguous(),
                dirs.contiguous(), positions.contiguous())
        _lib.check(lib.hp_pointnerf_aggregate(device._ptr(args[0]), device._ptr(args[1]), R, K, device._ptr(args[2]),
                                              device._ptr(args[3]), device._ptr(args[4]), o, device._ptr(args[5]),
                                              device._ptr(self.features), device._ptr(self.w1), device._ptr(self.w2),
                                              device._ptr(self.b2), device._ptr(g), device._stream()))
        return g

    def head(self, g: torch.Tensor) -> torch.Tensor:
        """(sigma, r, g, b): f32 [R, 4] (hp_pointnerf_head)."""
        lib = _lib.load(require_device=True)
        R = int(g.shape[0])
        out = torch.empty((max(R, 1), 4), dtype=torch.float32, device=g.device)[:R]
        _lib.check(lib.hp_pointnerf_head(device._ptr(g), R, device._ptr(self.w3), device._ptr(self.b3),
                                         device._ptr(self.w4), device._ptr(self.b4), device._ptr(out),
                                         device._stream()))
        return out

    def __call__(self, samples, dirs, origin, positions):
        """samples: a sampler 11-tuple with emit_knn (device)."""
        r_off, r_t, knn_id, knn_w = samples[0], samples[2], samples[9], samples[10]
        sr = sample_rays(r_off)
        g = self.aggregate(knn_id, knn_w, sr, r_t, dirs, origin, positions)
        return self.head(g), g

    # ------------------------------------------------------------ fp32 reference
    def inputs_reference(self, knn_id, sample_ray, r_t, dirs, origin, positions) -> torch.Tensor:
        """The input rows in fp32 (the device builds the same values in fp32 and
        rounds them to bf16)."""
        R, K = knn_id.shape
        o = torch.as_tensor(np.asarray(origin, np.float64), device=knn_id.device)
        ray = sample_ray.long()
        xs = o[None, :] + r_t[:, None] * dirs[ray]                                  # f64 [R,3]
        ok = knn_id >= 0
        idc = knn_id.clamp(min=0)
        d = (positions[idc] - xs[:, None, :]).float()                              # [R,K,3]
        f = self.features.float()[idc]                                             # [R,K,32]
        pe = []
        for c in range(3):
            for l in range(4):
                a = math.pi * d[..., c] * float(1 << l)
                pe += [torch.sin(a), torch.cos(a)]
        x = torch.cat([f, torch.stack(pe, -1), d, torch.ones_like(d[..., :1]),
                       torch.zeros_like(d[..., :1]).expand(R, K, 4)], -1)
        return torch.where(ok[..., None], x, torch.zeros_like(x))

    def reference(self, knn_id, knn_w, sample_ray, r_t, dirs, origin, positions):
        """fp32 restatement of the device computation, rounding to bf16 where
        the device stores bf16 (the MMA operands); returns (out [R,4], g)."""
        bf = lambda t: t.to(torch.bfloat16).float()  # noqa: E731
        x = bf(self.inputs_reference(knn_id, sample_ray, r_t, dirs, origin, positions))
        h1 = bf(torch.relu(x @ self.w1.float().T))
        h2 = torch.relu(h1 @ self.w2.float().T + self.b2)
        g = bf((h2 * knn_w.float()[..., None]).sum(1))
        h3 = torch.relu(g @ self.w3.float().T + self.b3)
        o = h3 @ self.w4.T + self.b4
        out = torch.cat([torch.nn.functional.softplus(o[:, :1]), torch.sigmoid(o[:, 1:])], 1)
        return out, g


def render_step(mlp: PointNeRFMLP, samples, dirs, origin, positions, pixels, t_far, width, height,
                background=(0.0, 0.0, 0.0)):
    """Colour / depth of each pixel from the aggregated density and colour of
    its retained samples: alpha_j = 1 - exp(-sigma_j delta_j) with the
    renderer's deltas (next t - t, the last one repeated, t_far - t for a
    single sample), composited by hp_render's volume mode."""
    out, _ = mlp(samples, dirs, origin, positions)
    r_off, r_t = samples[0], samples[2]
    R = int(r_t.shape[0])
    sr = sample_rays(r_off).long()
    nxt = torch.empty_like(r_t)
    if R:
        nxt[:-1] = r_t[1:]
        nxt[-1] = r_t[-1]
    first = r_off[:-1][sr]
    last = r_off[1:][sr] - 1
    idx = torch.arange(R, device=r_t.device)
    delta = torch.where(idx < last, nxt - r_t, r_t - torch.where(idx > first, torch.roll(r_t, 1), r_t))
    single = last == first
    delta = torch.where(single, t_far[sr] - r_t, delta)
    sigma = out[:, 0].double()
    alpha = -torch.expm1(-sigma * delta)
    rgb = out[:, 1:].double().contiguous()
    lib = _lib.load(require_device=True)
    owner = torch.full((height * width,), -1, dtype=torch.int32, device=r_t.device)
    color = torch.zeros((height, width, 3), dtype=torch.float64, device=r_t.device)
    depth = torch.zeros((height, width), dtype=torch.float64, device=r_t.device)
    bg = (ctypes.c_double * 3)(*background)
    _lib.check(lib.hp_render(0, device._ptr(r_off), int(r_off.shape[0]) - 1, device._ptr(samples[1]),
                             device._ptr(r_t), device._ptr(samples[3]), device._ptr(alpha), device._ptr(rgb),
                             None, device._ptr(pixels), 2, device._ptr(t_far), 1, bg, int(width), int(height),
                             device._ptr(owner), device._ptr(color), device._ptr(depth), device._stream()))
    return color, depth, out
