"""The library's multi-view batch driver (pipeline.search_and_sample_views):
one resident cloud, one index per view (reference renderer.py:113-125 /
cli.py:127-162), every view's samples equal to the single-view call and to
the C oracle."""

import numpy as np
import pytest

import paper_2404_14044_b200 as hp
from oracle import oracle as orc
from paper_2404_14044_b200 import pipeline

pytestmark = pytest.mark.gpu


def _views(n=4, w=64, h=48):
    cloud = hp.generate_scene(hp.SceneSpec("parallel_planes", n=30_000, seed=2, plane_count=3, plane_gap=0.5,
                                           extent=3.0, noise=0.005))
    cams, cfgs = [], []
    for k in range(n):
        th = 2.0 * np.pi * k / n
        cam = hp.scene_camera(w, h, fov_deg=55, origin=(0.4 * np.cos(th), 0.4 * np.sin(th), 0.0),
                              target=(0.0, 0.0, 4.0))
        cams.append(cam)
        cfgs.append(hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.01 * (1 + k % 2)),
                                    hp.pixel_disc_radius(cam)))
    return cloud, cams, cfgs


def _oracle_view(cloud, cam, cfg, sc):
    dirs, pixels = hp.ray_grid(cam)
    m = dirs.shape[0]
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius, cfg.use_approx_radius)
    b = orc.build(cloud.positions, cam, cfg.pad)
    q = orc.query(b["table_start"], b["table_count"], b["slot_x"], b["slot_y"], b["slot_z"],
                  b["reordered_ids"], cam.width + 2 * cfg.pad, cfg.pad, pixels[:, 0], pixels[:, 1],
                  dirs, cam.origin, np.ones(m), np.full(m, 10.0), slopes, threads=8)
    return orc.sample(*q[:4], slopes, sc.k_neighbors, sc.beta * sc.beta, sc.gamma, True, sc.epsilon,
                      sc.tau_min, cloud.colors, threads=8)


def test_views_equal_single_view_and_oracle():
    cloud, cams, cfgs = _views()
    sc = hp.SamplerConfig()
    got = pipeline.search_and_sample_views(cloud, cams, cfgs, 1.0, 10.0, sc)
    assert sorted(got) == list(range(len(cams)))
    for i, (cam, cfg) in enumerate(zip(cams, cfgs)):
        one = pipeline.search_and_sample_view(cloud, cam, cfg, 1.0, 10.0, sc)
        ref = _oracle_view(cloud, cam, cfg, sc)
        assert len(ref[1]) > 0
        for k in range(9):
            np.testing.assert_array_equal(got[i][k], one[k])
        for k in range(5):
            np.testing.assert_array_equal(got[i][k], ref[k])
        for k in (5, 6, 7, 8):
            np.testing.assert_allclose(got[i][k], ref[k], rtol=1e-12, atol=1e-300)


def test_views_one_config_no_colours():
    cloud, cams, cfgs = _views(n=3, w=40, h=30)
    got = pipeline.search_and_sample_views(cloud, cams, cfgs[0], 1.0, 10.0, with_colors=False)
    for i, cam in enumerate(cams):
        one = pipeline.search_and_sample_view(cloud, cam, cfgs[0], 1.0, 10.0, with_colors=False)
        assert got[i][7].shape == (0, 3)
        for k in range(9):
            np.testing.assert_array_equal(got[i][k], one[k])


def test_views_config_count_mismatch():
    cloud, cams, cfgs = _views(n=2, w=16, h=12)
    with pytest.raises(ValueError):
        pipeline.search_and_sample_views(cloud, cams, cfgs[:1] * 3, 1.0, 10.0)
