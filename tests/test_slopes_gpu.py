"""Device search-radius slopes (hp_radius_slopes) vs the
reference's numpy ``radius_slopes`` (geometry.py:249-260): bit-identical for
every pixel of many cameras, both radius formulas, grid rows and explicit
(strided) pixel arrays.  The device restates glibc's hypot, which is not
correctly rounded, so these equalities exercise its exact operation order."""

import numpy as np
import pytest
import torch

import paper_2404_14044_b200 as hp
from paper_2404_14044_b200 import device as dv
from paper_2404_14044_b200.geometry import Camera
from test_ray_grid_gpu import _cameras

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", range(4))
@pytest.mark.parametrize("approx", [False, True])
def test_slopes_bit_identical_grid_and_pixels(k, approx):
    cam = list(_cameras())[k]
    _, pixels = hp.ray_grid(cam)
    for f in (0.3, 1.0, 2.7):
        kr = f * hp.pixel_disc_radius(cam)
        ref = hp.radius_slopes(cam, pixels, kr, approx)
        np.testing.assert_array_equal(dv.radius_slopes(cam, kr, approx).cpu().numpy(), ref)
        W = cam.width
        r0, rows = cam.height // 3, max(cam.height // 2, 1)
        got = dv.radius_slopes(cam, kr, approx, row0=r0, m=rows * W).cpu().numpy()
        np.testing.assert_array_equal(got, ref[r0 * W:(r0 + rows) * W])
        px = torch.from_numpy(pixels).cuda()
        np.testing.assert_array_equal(dv.radius_slopes(cam, kr, approx, pixels=px).cpu().numpy(), ref)
        np.testing.assert_array_equal(dv.radius_slopes(cam, kr, approx, pixels=px[::3]).cpu().numpy(), ref[::3])


def test_slopes_random_cameras():
    """~3M slopes over random cameras (the reference's C2 parameter ranges)."""
    rng = np.random.default_rng(7)
    total = 0
    for _ in range(150):
        f = rng.uniform(0.5, 2.5)
        pw, ph = rng.uniform(5e-4, 5e-3), rng.uniform(5e-4, 5e-3)
        w, h = int(rng.integers(8, 257)), int(rng.integers(8, 257))
        cam = Camera.from_vectors((0, 0, 0), (0, 0, 1), (0, 1, 0), f, w, h, pw, ph)
        kr = rng.uniform(0.1, 4.0) * hp.pixel_disc_radius(cam)
        _, pixels = hp.ray_grid(cam)
        ref = hp.radius_slopes(cam, pixels, kr)
        np.testing.assert_array_equal(dv.radius_slopes(cam, kr).cpu().numpy(), ref)
        total += ref.size
    assert total > 1_000_000


def test_slopes_empty_and_errors():
    cam = hp.scene_camera(16, 12)
    assert dv.radius_slopes(cam, 0.01, m=0).numel() == 0
    with pytest.raises(ValueError):
        dv.radius_slopes(cam, 0.01, row0=5, m=16 * 12)  # past the grid
