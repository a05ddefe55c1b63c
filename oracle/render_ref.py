"""CPU restatement of the reference renderer over retained samples.

TEST INFRASTRUCTURE ONLY (the checker): imported by tests/ alone, never by the
package.  Restates, over the 9-tuple of sample_batch_arrays:
  * render_volume   reference renderer.py:163-185 (+ volume_sample_weights
                    :72-110: per-sample densities, deltas from np.diff, the
                    last delta repeated, t_far - t for a single sample);
  * render_knp      reference renderer.py:138-160 (k smallest perpendicular
                    distances by np.argpartition, inverse-distance weights or
                    the on-ray points alone, normalised);
  * _blank          reference renderer.py:128-135 (background, far plane of
                    the first ray).
Pinned: tests/test_render.py checks it against tests/golden/render_*.npz,
written by oracle/make_render_golden.py from the reference itself.
"""

from __future__ import annotations

import math

import numpy as np


def _deltas(ts, t_far):
    n = ts.shape[0]
    if n == 1:
        return np.array([t_far - ts[0]])
    d = np.empty(n)
    d[:-1] = np.diff(ts)
    d[-1] = d[-2]
    return d


def volume_weights(alphas, ts, t_far):
    """(weights, final transmittance) of one ray's retained samples."""
    n = alphas.shape[0]
    w = np.zeros(n)
    trans = 1.0
    if n == 0:
        return w, trans
    for j, (a, dt) in enumerate(zip(alphas.tolist(), _deltas(ts, t_far).tolist())):
        if a >= 1.0:
            absorbed, passed = 1.0, 0.0
        elif dt > 0.0:
            sigma = -math.log1p(-a) / dt
            passed = math.exp(-sigma * dt)
            absorbed = 1.0 - passed
        else:  # zero-length segment: the confidence itself
            absorbed, passed = a, 1.0 - a
        w[j] = trans * absorbed
        trans *= passed
    return w, trans


def render(mode, width, height, pixels, t_far, samples, point_colors, background, knp_k):
    """(color (H, W, 3), depth (H, W)) of the rays (pixels [m,2], t_far [m])."""
    r_off, r_id, r_t, r_dist, _, r_alpha, _, r_color, _ = samples
    m = pixels.shape[0]
    color = np.empty((height, width, 3))
    color[:, :] = background
    depth = np.full((height, width), float(t_far[0]) if m else 2.0)
    bg = np.asarray(background, dtype=np.float64)
    for i in range(m):
        lo, hi = int(r_off[i]), int(r_off[i + 1])
        u, v = int(pixels[i, 0]), int(pixels[i, 1])
        if mode == "volume":
            if hi == lo:
                color[v, u] = bg
                depth[v, u] = t_far[i]
                continue
            w, trans = volume_weights(r_alpha[lo:hi], r_t[lo:hi], float(t_far[i]))
            color[v, u] = w @ r_color[lo:hi] + trans * bg
            s = float(w.sum())
            depth[v, u] = float(w @ r_t[lo:hi]) / s if s > 0 else t_far[i]
        else:
            if hi == lo:
                continue
            d = r_dist[lo:hi]
            k = min(knp_k, hi - lo)
            pick = np.argpartition(d, k - 1)[:k]
            dk = d[pick]
            on_ray = dk == 0.0
            w = on_ray.astype(np.float64) if on_ray.any() else 1.0 / dk
            w /= w.sum()
            color[v, u] = w @ point_colors[r_id[lo:hi][pick]]
            depth[v, u] = float(w @ r_t[lo:hi][pick])
    return color, depth


def knp_tie_rays(samples, knp_k):
    """Rays whose k-th smallest distance is tied with the next one (the
    selected set, hence the colour, depends on the tie order)."""
    r_off, r_dist = samples[0], samples[3]
    out = []
    for i in range(r_off.shape[0] - 1):
        d = np.sort(r_dist[r_off[i]:r_off[i + 1]])
        k = min(knp_k, d.shape[0])
        if 0 < k < d.shape[0] and d[k - 1] == d[k]:
            out.append(i)
    return np.array(out, dtype=np.int64)
