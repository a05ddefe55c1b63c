"""The reference's host-side acceptance criteria (CPU, no GPU needed).

Ports /root/reference/pkg/tests/test_acceptance.py C2 (126-176, the search
radius formulas: the scalar ``radius_slope`` and the library's host-thread
``hp_radius_slopes_host`` that feeds the device path, against a 50-digit
evaluation) and C3 (179-203, occlusion-weight algebra).  The GPU criteria are
in test_acceptance_gpu.py.
"""

import math

import mpmath
import numpy as np

from paper_2404_14044_b200.geometry import (Camera, pixel_disc_radius, radius_slope,
                                            radius_slopes)
from paper_2404_14044_b200.pipeline import host_slopes
from paper_2404_14044_b200.sampler import SampleCandidate, occlusion_weights


def test_c2_radius_formulas():
    """Exact radius vs 50-digit evaluation; small-angle bound for the approximation."""
    rng = np.random.default_rng(7)
    worst_exact = 0.0
    for _ in range(1000):
        f = rng.uniform(0.5, 2.5)
        pw = rng.uniform(5e-4, 5e-3)
        ph = rng.uniform(5e-4, 5e-3)
        w = int(rng.integers(8, 257))
        h = int(rng.integers(8, 257))
        cam = Camera.from_vectors((0, 0, 0), (0, 0, 1), (0, 1, 0), f, w, h, pw, ph)
        u = int(rng.integers(0, w))
        v = int(rng.integers(0, h))
        kr = rng.uniform(0.1, 4.0) * pixel_disc_radius(cam)
        t = rng.uniform(0.5, 20.0)
        px = np.array([[u, v]], np.int64)
        lib = host_slopes(cam, px, kr, threads=1)
        assert np.array_equal(lib, radius_slopes(cam, px, kr))  # bit-identical to numpy
        with mpmath.workdps(50):
            du = (mpmath.mpf(u) + mpmath.mpf("0.5") - mpmath.mpf(w) / 2) * mpmath.mpf(pw)
            dv = (mpmath.mpf(v) + mpmath.mpf("0.5") - mpmath.mpf(h) / 2) * mpmath.mpf(ph)
            mf = mpmath.mpf(f)
            ae = mpmath.sqrt(mf * mf + du * du + dv * dv)
            ge = mpmath.sqrt(ae * ae - mf * mf)
            ab = mpmath.sqrt((ge - mpmath.mpf(kr)) ** 2 + mf * mf)
            expected = float(mpmath.mpf(t) * mf * mpmath.mpf(kr) / (ae * ab))
        for got in (t * radius_slope(cam, (u, v), kr), t * float(lib[0])):
            worst_exact = max(worst_exact, abs(got - expected) / expected)
    assert worst_exact <= 1e-12

    worst_approx = 0.0
    one_degree = math.radians(1.0)
    for _ in range(1000):
        f = rng.uniform(1.0, 2.0)
        pix = rng.uniform(1e-3, 2e-3)
        w = int(rng.integers(32, 97))
        h = int(rng.integers(32, 97))
        cam = Camera.from_vectors((0, 0, 0), (0, 0, 1), (0, 1, 0), f, w, h, pix, pix)
        u = int(rng.integers(0, w))
        v = int(rng.integers(0, h))
        kr = rng.uniform(0.5, 2.0) * pixel_disc_radius(cam)
        du = (u + 0.5 - 0.5 * w) * pix
        dv = (v + 0.5 - 0.5 * h) * pix
        ae = math.sqrt(f * f + du * du + dv * dv)
        assert math.atan(kr / ae) < one_degree
        t = rng.uniform(0.5, 10.0) * f
        exact = t * radius_slope(cam, (u, v), kr, approx=False)
        approx = t * radius_slope(cam, (u, v), kr, approx=True)
        px = np.array([[u, v]], np.int64)
        assert np.array_equal(host_slopes(cam, px, kr, approx=True, threads=1),
                              radius_slopes(cam, px, kr, approx=True))
        worst_approx = max(worst_approx, abs(approx - exact) / exact)
    assert worst_approx <= 1e-3


def test_c3_weight_algebra():
    """Occlusion weights match naive products; the weight sum telescopes."""
    rng = np.random.default_rng(11)
    worst = worst_sum = 0.0
    for _ in range(10_000):
        alphas = rng.uniform(0.0, 1.0, int(rng.integers(1, 21)))
        cands = [SampleCandidate(t=float(j), position=np.zeros(3), radius=1.0,
                                 dist_perp=0.0, point_id=j) for j in range(alphas.size)]
        for c, a in zip(cands, alphas):
            c.confidence = float(a)
        occlusion_weights(cands)
        trans = 1.0
        for j, c in enumerate(cands):
            worst = max(worst, abs(c.weight - alphas[j] * math.prod(1.0 - alphas[:j])))
            trans *= 1.0 - alphas[j]
        worst_sum = max(worst_sum, abs(sum(c.weight for c in cands) - (1.0 - trans)))
    assert worst <= 1e-12
    assert worst_sum <= 1e-9
