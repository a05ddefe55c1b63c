"""hp_build_layout (the query layout alone, optionally for a row window):
the same row pointers and per-pixel point sets as the full build's layout
(the order inside a pixel is free), bit-identical coordinates; a row window
keeps exactly the points of those padded rows; frames over a row band give
the same samples with the band-restricted index."""
import numpy as np
import pytest
import torch

import golden_util as gu
import paper_2404_14044_b200 as hp
from paper_2404_14044_b200 import device as dv
from paper_2404_14044_b200 import pipeline

pytestmark = pytest.mark.gpu


def _pixel_sets(idx, n_in):
    rp = idx.row_ptr.cpu().numpy()
    pid = idx.point_id[:n_in].cpu().numpy()
    r4 = idx.rel4[:n_in].cpu().numpy()
    order = np.lexsort((pid, np.repeat(np.arange(len(rp) - 1), np.diff(rp))))
    return rp, pid[order], r4[order]


@pytest.mark.parametrize("name", ["cfg1", "small_sphere_surface", "orbit_planes"])
def test_layout_build_matches_full_build(name):
    if name not in gu.case_names():
        pytest.skip(f"no golden case {name}")
    _, cloud, cam, cfg, *_ = gu.get_case(name)
    dev = torch.device("cuda")
    xyz = torch.from_numpy(np.array(cloud.positions)).to(dev)
    full = dv.build(xyz, cam, cfg.pad)
    lay = dv.build_layout(xyz, cam, cfg.pad)
    assert lay.n_in == full.n_in and lay.table_start is None
    a, b = _pixel_sets(full, full.n_in), _pixel_sets(lay, lay.n_in)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    # a row window: exactly the points of padded rows [a, b + 2 pad)
    H = cam.height
    r0, r1 = H // 3, H // 2
    win = dv.build_layout(xyz, cam, cfg.pad, rows=(r0, r1))
    wp = full.padded_width
    rp = a[0]
    lo, hi = rp[r0 * wp], rp[min(r1 + 2 * cfg.pad, full.padded_height) * wp]
    assert win.n_in == hi - lo
    np.testing.assert_array_equal(np.diff(win.row_ptr.cpu().numpy())[r0 * wp:(r1 + 2 * cfg.pad) * wp],
                                  np.diff(rp)[r0 * wp:(r1 + 2 * cfg.pad) * wp])


def test_band_frame_with_row_window_equals_whole_index():
    cloud = hp.generate_scene(hp.SceneSpec("sphere_surface", n=60_000, seed=2, noise=0.005))
    cam = hp.scene_camera(160, 120, fov_deg=30)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.01), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    W = cam.width
    a, b = 40 * W, 70 * W  # image rows [40, 70)
    slopes = hp.radius_slopes(cam, pixels[a:b], cfg.kernel_radius)
    dev = torch.device("cuda")
    up = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    xyz, col = up(cloud.positions), up(cloud.colors)
    rays = (up(pixels[a:b]), up(dirs[a:b]), up(np.full(b - a, 1.0)), up(np.full(b - a, 10.0)), up(slopes))
    whole = pipeline.frame_device(xyz, col, cam, cfg, *rays, hp.SamplerConfig(), True)
    band = pipeline.frame_device(xyz, col, cam, cfg, *rays, hp.SamplerConfig(), True, rows=(40, 70))
    assert band.index.n_in < whole.index.n_in
    for x, y in zip(whole.samples, band.samples):
        assert torch.equal(x, y)
    assert band.R > 0


def test_distributed_view_single_rank_equals_view(tmp_path):
    """shard.search_and_sample_distributed on a one-rank group: the layout
    build's per-pixel counts give the (single) band, and the result equals
    search_and_sample_view's arrays."""
    import torch.distributed as dist

    from paper_2404_14044_b200 import shard
    cloud = hp.generate_scene(hp.SceneSpec("sphere_surface", n=40_000, seed=4, noise=0.005))
    cam = hp.scene_camera(120, 90, fov_deg=30)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.01), hp.pixel_disc_radius(cam))
    init = not dist.is_initialized()
    if init:
        dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    try:
        got = shard.search_and_sample_distributed(cloud, cam, cfg, 1.0, 10.0, dist)
    finally:
        if init:
            dist.destroy_process_group()
    ref = pipeline.search_and_sample_view(cloud, cam, cfg, 1.0, 10.0)
    assert len(got) == len(ref)
    for x, y in zip(got, ref):
        np.testing.assert_array_equal(x, y)
    assert ref[1].size > 0
