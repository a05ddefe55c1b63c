"""On-device ray grid (hp_ray_grid) vs the reference's
numpy ``ray_grid`` (geometry.py:289-306): bit-identical directions and pixels
for look-at and rotated off-origin cameras, odd sizes and non-square pixels,
whole images and row ranges; and the whole-view pipeline
(``search_and_sample_view``) equal to ``search_and_sample`` on host rays."""

import numpy as np
import pytest
import torch

import paper_2404_14044_b200 as hp
from paper_2404_14044_b200 import device as dv
from paper_2404_14044_b200 import pipeline
from paper_2404_14044_b200.geometry import Camera

pytestmark = pytest.mark.gpu


def _cameras():
    yield hp.scene_camera(200, 200, fov_deg=40)
    yield hp.scene_camera(640, 480, fov_deg=60, origin=(0.4 * np.cos(1.3), 0.4 * np.sin(1.3), 0.0),
                          target=(0.0, 0.0, 4.0))
    yield hp.scene_camera(37, 23, fov_deg=73, origin=(0.3, -0.2, 0.1), target=(1.0, 2.0, 5.0),
                          up=(0.2, 1.0, 0.1), focal_length=1.7)
    yield Camera.from_vectors(np.array([1.0, -2.0, 0.5]), np.array([0.3, 0.9, 1.0]), (0.0, 0.0, 1.0),
                              2.5, 41, 17, 0.0123, 0.0171)


@pytest.mark.parametrize("k", range(4))
def test_ray_grid_bit_identical(k):
    cam = list(_cameras())[k]
    dirs, pixels = hp.ray_grid(cam)
    d, p, tn, tf = dv.ray_grid(cam, t_near=1.0, t_far=10.0)
    np.testing.assert_array_equal(d.cpu().numpy(), dirs)
    np.testing.assert_array_equal(p.cpu().numpy(), pixels)
    assert torch.all(tn == 1.0) and torch.all(tf == 10.0)
    W = cam.width
    r0, rows = cam.height // 3, cam.height // 2
    d2, p2, _, _ = dv.ray_grid(cam, row0=r0, rows=rows)
    np.testing.assert_array_equal(d2.cpu().numpy(), dirs[r0 * W:(r0 + rows) * W])
    np.testing.assert_array_equal(p2.cpu().numpy(), pixels[r0 * W:(r0 + rows) * W])


def test_view_pipeline_equals_host_rays():
    cloud = hp.generate_scene(hp.SceneSpec("sphere_surface", n=100_000, seed=0, noise=0.005))
    cam = hp.scene_camera(200, 200, fov_deg=40)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.01), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    m = dirs.shape[0]
    a = pipeline.search_and_sample_view(cloud, cam, cfg, 1.0, 10.0)
    b = pipeline.search_and_sample(cloud, cam, cfg, pixels, dirs, np.full(m, 1.0), np.full(m, 10.0))
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    assert a[1].size > 0


@pytest.mark.parametrize("chunks", [2, 5])
def test_chunked_host_copies_equal_one_pass(chunks, monkeypatch):
    """Ray chunks with overlapped result copies (pipeline._samples_to_host)
    give the one-pass arrays -- also when the host buffers sized from the
    first chunk are short and grow mid-frame."""
    cloud = hp.generate_scene(hp.SceneSpec("sphere_surface", n=50_000, seed=3, noise=0.005))
    cam = hp.scene_camera(160, 120, fov_deg=25)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.01), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    m = dirs.shape[0]
    monkeypatch.setattr(pipeline, "E2E_CUTS", ())
    ref = pipeline.search_and_sample(cloud, cam, cfg, pixels, dirs, np.full(m, 1.0), np.full(m, 10.0))
    monkeypatch.setattr(pipeline, "E2E_CUTS", tuple(k / chunks for k in range(1, chunks)))
    monkeypatch.setattr(pipeline, "E2E_MIN_RAYS", 1)
    monkeypatch.setattr(pipeline, "E2E_HEADROOM", 0.5)  # the first guess is short: the buffers grow
    for view in (False, True):
        pipeline._R_PER_RAY.clear()  # no size hint from an earlier frame
        out = (pipeline.search_and_sample_view(cloud, cam, cfg, 1.0, 10.0) if view else
               pipeline.search_and_sample(cloud, cam, cfg, pixels, dirs, 1.0, 10.0))
        assert len(out) == len(ref)
        for x, y in zip(out, ref):
            np.testing.assert_array_equal(x, y)
