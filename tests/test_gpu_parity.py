"""Device path (sm_100a kernels through the C ABI) vs the reference goldens and
the C oracle.  Bit-exact for ids/offsets/tables/t/dist/udf and the primary
surface point; alpha / w / colour / t_end within golden_util.VAL_RTOL (the
device exp() may differ from glibc's by an ulp; north_star's bar is 1e-5)."""

import numpy as np
import pytest
import torch

import golden_util as gu
from oracle import oracle as orc
from paper_2404_14044_b200 import device as dv

pytestmark = pytest.mark.gpu


def _dev_case(name):
    _, cloud, cam, cfg, tn, tf, stride, samplers = gu.get_case(name)
    dev = torch.device("cuda")
    idx = dv.build(torch.from_numpy(cloud.positions).to(dev), cam, cfg.pad)
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rays = (up(pixels), up(dirs), up(t_near), up(t_far), up(slopes))
    return cloud, cam, cfg, samplers, idx, rays


@pytest.mark.parametrize("name", gu.case_names())
def test_build_bit_exact(name):
    g = gu.load(name)
    cloud, cam, cfg, samplers, idx, rays = _dev_case(name)
    for k in gu.BUILD_FIELDS:
        assert gu.digest(getattr(idx, k).cpu().numpy()) == g[f"build_{k}_sha"], f"build {k}"
    assert idx.n_in == int(np.count_nonzero(orc.rasterize(cloud.positions, cam, cfg.pad) >= 0))


@pytest.mark.parametrize("name", gu.case_names())
def test_query_bit_exact(name):
    g = gu.load(name)
    cloud, cam, cfg, samplers, idx, rays = _dev_case(name)
    q = [x.cpu().numpy() for x in dv.query(idx, *rays)]
    for k, v in zip(gu.QUERY_FIELDS, q):
        assert gu.digest(v) == g[f"query_{k}_sha"], f"query {k}"


@pytest.mark.parametrize("name", gu.case_names())
@pytest.mark.parametrize("exact_t_end", [True, False])
def test_sample_matches_reference(name, exact_t_end):
    g = gu.load(name)
    cloud, cam, cfg, samplers, idx, rays = _dev_case(name)
    q = dv.query(idx, *rays)
    colors = torch.from_numpy(cloud.colors).cuda()
    for sname in samplers:
        sc = gu.sampler_config(sname)
        for colored in ((True, False) if sname == "default" else (True,)):
            out = dv.sample(q[0], q[1], q[2], q[3], rays[4], sc, colors if colored else None,
                            exact_t_end=exact_t_end)
            out = [x.cpu().numpy() for x in out]
            tag = f"sample_{sname}{'' if colored else '_nocolor'}_"
            gu.check_sample(g, tag, out, g["rows"], check_t_end=exact_t_end)
            pid, pt = dv.primary_surface(*[torch.from_numpy(a).cuda() for a in (out[0], out[1], out[2])])
            assert gu.digest(pid.cpu().numpy()) == g[tag + "primary_sha"]


def test_layout_from_reference_table_equals_build():
    name = "small_parallel_planes"
    g = gu.load(name)
    cloud, cam, cfg, samplers, idx, rays = _dev_case(name)
    t = lambda k: torch.from_numpy(g[f"build_{k}"]).cuda()  # noqa: E731
    idx2 = dv.build_from_table(t("table_start"), t("table_count"), t("slot_x"), t("slot_y"),
                               t("slot_z"), t("reordered_ids"), cam, cfg.pad)
    for k in ("row_ptr", "rel_x", "rel_y", "rel_z", "point_id"):
        assert torch.equal(getattr(idx2, k)[: idx.n_in + (1 if k == "row_ptr" else 0)],
                           getattr(idx, k)[: idx.n_in + (1 if k == "row_ptr" else 0)]), k
    q1 = dv.query(idx, *rays)
    q2 = dv.query(idx2, *rays)
    for a, b in zip(q1, q2):
        assert torch.equal(a, b)


@pytest.mark.parametrize("name", gu.case_names())
def test_cone_footprint_is_transparent(name):
    """Testing only footprint pixels gives exactly the full-window result."""
    cloud, cam, cfg, samplers, idx, rays = _dev_case(name)
    a = dv.query(idx, *rays, footprint=True)
    b = dv.query(idx, *rays, footprint=False)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


def test_footprint_on_wide_rotated_camera():
    """Wide field of view, rotated off-origin camera, large delta."""
    import paper_2404_14044_b200 as hp
    cloud = hp.generate_scene(hp.SceneSpec("uniform_box", n=40_000, seed=8, extent=3.0))
    cam = hp.scene_camera(96, 64, fov_deg=110, origin=(0.7, -0.4, 0.3), target=(0.2, 0.1, 4.0),
                          up=(0.3, 1.0, 0.1))
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.05), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    m = dirs.shape[0]
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
    dev = torch.device("cuda")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    idx = dv.build(up(cloud.positions), cam, cfg.pad)
    rays = (up(pixels), up(dirs), up(np.full(m, 0.5)), up(np.full(m, 9.0)), up(slopes))
    a = dv.query(idx, *rays, footprint=True)
    b = dv.query(idx, *rays, footprint=False)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    ob = orc.build(cloud.positions, cam, cfg.pad)
    oq = orc.query(ob["table_start"], ob["table_count"], ob["slot_x"], ob["slot_y"], ob["slot_z"],
                   ob["reordered_ids"], cam.width + 2 * cfg.pad, cfg.pad, pixels[:, 0], pixels[:, 1],
                   dirs, cam.origin, np.full(m, 0.5), np.full(m, 9.0), slopes)
    for x, y in zip(a, oq):
        np.testing.assert_array_equal(x.cpu().numpy(), y)


@pytest.mark.parametrize("name", gu.case_names())
@pytest.mark.parametrize("exact_t_end", [True, False])
def test_query_facts_do_not_change_samples(name, exact_t_end):
    """The sampler's fast path fed by the query's per-ray facts gives the
    same arrays as the sampler computing its own preconditions."""
    cloud, cam, cfg, samplers, idx, rays = _dev_case(name)
    q = dv.query(idx, *rays, facts=True)
    assert all(torch.equal(a, b) for a, b in zip(q[:6], dv.query(idx, *rays)))
    colors = torch.from_numpy(cloud.colors).cuda()
    for sname in samplers:
        sc = gu.sampler_config(sname)
        a = dv.sample(q[0], q[1], q[2], q[3], rays[4], sc, colors, exact_t_end=exact_t_end, facts=q[6])
        b = dv.sample(q[0], q[1], q[2], q[3], rays[4], sc, colors, exact_t_end=exact_t_end)
        for x, y in zip(a, b):
            assert torch.equal(x, y)


def test_ray_chunked_frame_equals_single_pass():
    """pipeline.frame_device split into ray chunks (match budget forced
    small) returns exactly the single-pass samples."""
    import paper_2404_14044_b200 as hp
    from paper_2404_14044_b200 import pipeline
    cloud = hp.generate_scene(hp.SceneSpec("sphere_surface", n=60_000, seed=2, noise=0.005))
    cam = hp.scene_camera(96, 80, fov_deg=40)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.01), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    m = dirs.shape[0]
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    args = (up(cloud.positions), up(cloud.colors), cam, cfg, up(pixels), up(dirs), up(np.full(m, 1.0)),
            up(np.full(m, 10.0)), up(slopes))
    one = pipeline.frame_device(*args)
    assert one.chunks == 1
    many = pipeline.frame_device(*args, max_matches=max(one.Q // 7, 1))
    assert many.chunks >= 7 and many.Q == one.Q and many.query is None
    for a, b in zip(one.samples, many.samples):
        assert torch.equal(a, b)


def test_degenerate_frames():
    """No rays, rays that hit nothing, an empty cloud: the chained device
    path returns empty / all-zero results without launching garbage."""
    import paper_2404_14044_b200 as hp
    from paper_2404_14044_b200 import pipeline
    cam = hp.scene_camera(16, 12, fov_deg=40)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.01), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    far = hp.generate_scene(hp.SceneSpec("uniform_box", n=500, seed=1, center=(0.0, 0.0, 50.0), extent=1.0))
    empty = np.zeros((0, 3))
    for pos, m in ((far.positions, dirs.shape[0]), (empty, dirs.shape[0]), (far.positions, 0)):
        fr = pipeline.frame_device(up(pos), None, cam, cfg, up(pixels[:m]), up(dirs[:m]),
                                   up(np.full(m, 1.0)), up(np.full(m, 10.0)), up(slopes[:m]))
        r_off, r_id, *_, t_end = fr.samples
        assert fr.Q == 0 and r_id.numel() == 0 and r_off.numel() == m + 1
        assert torch.all(r_off == 0) and torch.all(t_end == 1.0)


@pytest.mark.parametrize("name", ["cfg1", "small_sphere_surface", "orbit_planes", "empty"])
@pytest.mark.parametrize("mode", [None, True, False])
@pytest.mark.parametrize("chunks", [1, 3])
def test_search_and_sample_host_api_matches_goldens(name, mode, chunks, monkeypatch):
    """The public host-buffer pipeline (numpy in / numpy out, side-stream
    uploads, host slopes in the library, ray chunks whose copies overlap the
    neighbouring chunks' work) reproduces the reference goldens in every
    frame mode (auto, prefix, full CSR)."""
    from paper_2404_14044_b200 import pipeline
    if name not in gu.case_names():
        pytest.skip(f"no golden case {name}")
    monkeypatch.setattr(pipeline, "PREFIX", mode)
    monkeypatch.setattr(pipeline, "E2E_CUTS", tuple(k / chunks for k in range(1, chunks)))
    monkeypatch.setattr(pipeline, "E2E_MIN_RAYS", 1)
    g = gu.load(name)
    _, cloud, cam, cfg, tn, tf, stride, samplers = gu.get_case(name)
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    out = pipeline.search_and_sample(cloud, cam, cfg, pixels, dirs, t_near, t_far)
    gu.check_sample(g, "sample_default_", out, g["rows"], check_t_end=True)
