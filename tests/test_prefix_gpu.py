"""hp_head_count + hp_head_sort: each ray's head is exactly the first
``plen`` entries of the full (t, id)-sorted CSR (bit for bit), it is closed
under t (the next match has a strictly larger t), the cuts are lower bounds
of every left-out match's t and dist, and the sampler facts (counted over
the head) equal the full query's when the head is the whole segment and
never exceed them otherwise.

Reference behaviour being preserved: _kernels.hash_query_batch
(_kernels.py:86-157) sorts every ray's matches by (t, id); a prefix of that
order is what _kernels.sample_batch (_kernels.py:552-700) walks first.
"""

import numpy as np
import pytest
import torch

import golden_util as gu
import paper_2404_14044_b200 as hp
from paper_2404_14044_b200 import device as dv

pytestmark = pytest.mark.gpu


def _check_prefix(q, p, want):
    off = q[0].cpu().numpy()
    ids, t, d = (x.cpu().numpy() for x in q[1:4])
    fa = q[6].cpu().numpy()
    np.testing.assert_array_equal(p.offsets.cpu().numpy(), off)
    start = p.start.cpu().numpy()
    plen = p.length.cpu().numpy()
    pf = p.facts.cpu().numpy()
    whole = plen == np.diff(off)  # facts over the prefix: the full ones when it is everything
    np.testing.assert_array_equal(pf[whole], fa[whole])
    assert np.all((pf[~whole] <= fa[~whole]) | (plen[~whole] == 0))
    pt, pid, pd = p.t.cpu().numpy(), p.ids.cpu().numpy(), p.dist.cpu().numpy()
    ct, cd = p.cut_t.cpu().numpy(), p.cut_d.cpu().numpy()
    counts = np.diff(off)
    assert np.all(plen <= counts)
    short = plen < np.minimum(counts, want)
    for r in np.flatnonzero(counts):
        a, n, s = off[r], plen[r], start[r]
        np.testing.assert_array_equal(pt[s:s + n], t[a:a + n])
        np.testing.assert_array_equal(pid[s:s + n].astype(np.int64), ids[a:a + n])
        np.testing.assert_array_equal(pd[s:s + n], d[a:a + n])
        if n < counts[r] and n > 0:
            assert t[a + n] > t[a + n - 1]
        rest = slice(a + n, a + counts[r])
        if n < counts[r]:  # lower bounds of the left-out matches
            assert np.all(t[rest] >= ct[r]) and np.all(d[rest] >= cd[r])
            assert n == 0 or ct[r] > t[a + n - 1]
        else:
            assert ct[r] == np.inf and cd[r] == np.inf
        if short[r]:  # only when a single selection bin holds more than the cap
            assert n < want
    return plen, counts


@pytest.mark.parametrize("name", gu.case_names())
@pytest.mark.parametrize("want", [1, 7, 64, 512])
@pytest.mark.parametrize("whole", ["want", 1024])
def test_prefix_is_the_sorted_csr_head(name, want, whole):
    _, cloud, cam, cfg, tn, tf, stride, _ = gu.get_case(name)
    dev = torch.device("cuda")
    idx = dv.build(torch.from_numpy(cloud.positions).to(dev), cam, cfg.pad)
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rays = (up(pixels), up(dirs), up(t_near), up(t_far), up(slopes))
    q = dv.query(idx, *rays, facts=True)
    p = dv.query_prefix(idx, *rays, want=want, whole=want if whole == "want" else whole)
    _check_prefix(q, p, want)


def test_prefix_on_dense_rays():
    """q up to thousands per ray: the prefix is selected by histogram, not
    the whole segment."""
    cloud = hp.generate_scene(hp.SceneSpec("parallel_planes", n=60_000, seed=3, plane_count=3,
                                           plane_gap=0.05, extent=0.8, noise=0.01))
    cam = hp.scene_camera(48, 40, fov_deg=14)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.04), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    dirs, pixels = dirs[::11], pixels[::11]
    tn, tf = np.full(len(dirs), 1.0), np.full(len(dirs), 10.0)
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
    dev = torch.device("cuda")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    idx = dv.build(up(cloud.positions), cam, cfg.pad)
    rays = (up(pixels), up(dirs), up(tn), up(tf), up(slopes))
    q = dv.query(idx, *rays, facts=True)
    for want, whole in ((16, 16), (16, 1024), (300, 300), (300, 640), (700, 700)):
        p = dv.query_prefix(idx, *rays, want=want, whole=whole)
        plen, counts = _check_prefix(q, p, want)
        assert (counts > want).sum() > 10
        # the head reaches ~want (a trim at the key cut may leave it a little short)
        assert np.mean(plen[counts > want] >= 0.75 * want) > 0.9


def _prefix_frame(idx, rays, sc, colors, exact_t_end, want, whole=None, factors=False):
    """prefix-mode sampling with the flagged rays re-run on the full path
    (``factors``: the heads carry precomputed bound factors)"""
    pre = dv.query_prefix(idx, *rays, want=want, whole=whole, sampler_cfg=sc if factors else None)
    *s, flagged, n_flagged = dv.sample_prefix(pre, rays[4], sc, colors, exact_t_end)
    fl = flagged.cpu().numpy()
    assert int((fl != 0).sum()) == n_flagged
    cnt = np.diff(s[0].cpu().numpy())
    assert np.all(cnt[fl != 0] == 0)
    if n_flagged:
        sel = torch.nonzero(flagged, as_tuple=True)[0]
        q = dv.query(idx, *[r[sel] for r in rays], facts=True)
        sub = dv.sample(q[0], q[1], q[2], q[3], rays[4][sel], sc, colors, exact_t_end, facts=q[6])
        s = dv.merge_flagged(tuple(s), flagged, sub)
    return s, n_flagged


def _assert_same(a, b):
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x.cpu().numpy(), y.cpu().numpy())


@pytest.mark.parametrize("name", gu.case_names())
@pytest.mark.parametrize("exact_t_end", [True, False])
@pytest.mark.parametrize("want", [1, 9, 512])
@pytest.mark.parametrize("whole", ["want", 1024])
@pytest.mark.parametrize("factors", [False, True])
def test_prefix_sampling_equals_full(name, exact_t_end, want, whole, factors):
    _, cloud, cam, cfg, tn, tf, stride, samplers = gu.get_case(name)
    dev = torch.device("cuda")
    idx = dv.build(torch.from_numpy(cloud.positions).to(dev), cam, cfg.pad)
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rays = (up(pixels), up(dirs), up(t_near), up(t_far), up(slopes))
    q = dv.query(idx, *rays, facts=True)
    colors = torch.from_numpy(cloud.colors).cuda()
    for sname in samplers:
        sc = gu.sampler_config(sname)
        for col in ((colors, None) if sname == "default" else (colors,)):
            full = dv.sample(q[0], q[1], q[2], q[3], rays[4], sc, col, exact_t_end=exact_t_end, facts=q[6])
            got, _ = _prefix_frame(idx, rays, sc, col, exact_t_end, want, want if whole == "want" else whole,
                                   factors)
            _assert_same(got, full)


@pytest.mark.parametrize("k,mode,gamma", [(8, "epsilon", 0.9), (40, "epsilon", 0.5), (3, "tau", 0.3)])
@pytest.mark.parametrize("exact_t_end", [True, False])
def test_prefix_sampling_on_dense_rays(k, mode, gamma, exact_t_end):
    cloud = hp.generate_scene(hp.SceneSpec("parallel_planes", n=60_000, seed=3, plane_count=3,
                                           plane_gap=0.05, extent=0.8, noise=0.01))
    cam = hp.scene_camera(48, 40, fov_deg=14)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.04), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    dirs, pixels = dirs[::5], pixels[::5]
    tn, tf = np.full(len(dirs), 1.0), np.full(len(dirs), 10.0)
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
    dev = torch.device("cuda")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    idx = dv.build(up(cloud.positions), cam, cfg.pad)
    rays = (up(pixels), up(dirs), up(tn), up(tf), up(slopes))
    q = dv.query(idx, *rays, facts=True)
    sc = hp.SamplerConfig(k_neighbors=k, retention_mode=mode, gamma=gamma)
    colors = torch.from_numpy(cloud.colors).cuda()
    full = dv.sample(q[0], q[1], q[2], q[3], rays[4], sc, colors, exact_t_end=exact_t_end, facts=q[6])
    seen = []
    for want, whole in ((16, 16), (16, 1024), (64, 64), (512, 512), (512, 1024)):
        for factors in (False, True):
            got, nf = _prefix_frame(idx, rays, sc, colors, exact_t_end, want, whole, factors)
            _assert_same(got, full)
        seen.append(nf)
    assert seen[0] > 0  # the small heads do send rays to the full path


@pytest.mark.parametrize("exact_t_end", [True, False])
def test_pipeline_prefix_frame_equals_full_frame(exact_t_end):
    from paper_2404_14044_b200 import pipeline
    _, cloud, cam, cfg, tn, tf, stride, _ = gu.get_case("cfg1")
    dev = torch.device("cuda")
    xyz = torch.from_numpy(cloud.positions).to(dev)
    col = torch.from_numpy(cloud.colors).to(dev)
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rays = (up(pixels), up(dirs), up(t_near), up(t_far), up(slopes))
    idx = dv.build(xyz, cam, cfg.pad)
    sc = hp.SamplerConfig()
    a = pipeline._query_sample(idx, col, *rays, sc, exact_t_end, None, prefix=True)
    b = pipeline._query_sample(idx, col, *rays, sc, exact_t_end, None, prefix=False)
    _assert_same(a.samples, b.samples)
    assert a.Q == b.Q


def test_pipeline_prefix_chunked_frame_equals_full_frame():
    """A frame over the match budget runs in ray chunks in prefix mode too."""
    from paper_2404_14044_b200 import pipeline
    _, cloud, cam, cfg, tn, tf, stride, _ = gu.get_case("cfg1")
    dev = torch.device("cuda")
    xyz = torch.from_numpy(cloud.positions).to(dev)
    col = torch.from_numpy(cloud.colors).to(dev)
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rays = (up(pixels), up(dirs), up(t_near), up(t_far), up(slopes))
    idx = dv.build(xyz, cam, cfg.pad)
    sc = hp.SamplerConfig()
    b = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=False)
    a = pipeline._query_sample(idx, col, *rays, sc, True, max(b.Q // 5, 4096), prefix=True)
    assert a.chunks > 1
    _assert_same(a.samples, b.samples)
    assert a.Q == b.Q


@pytest.mark.parametrize("want,whole", [(16, 16), (64, 1024), (400, 512)])
def test_pipeline_second_chance_resort_equals_full(monkeypatch, want, whole):
    """Short heads send many rays to the second chance (their heads re-sorted
    up to 1024 from the same count pass); the frame still equals the full-CSR
    frame, and only rays still flagged after that take the full path."""
    from paper_2404_14044_b200 import pipeline
    monkeypatch.setattr(dv, "PREFIX_WANT", want)
    monkeypatch.setattr(dv, "HEAD_WHOLE", whole)
    cloud = hp.generate_scene(hp.SceneSpec("parallel_planes", n=60_000, seed=3, plane_count=3,
                                           plane_gap=0.05, extent=0.8, noise=0.01))
    cam = hp.scene_camera(48, 40, fov_deg=14)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.04), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    tn, tf = np.full(len(dirs), 1.0), np.full(len(dirs), 10.0)
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
    dev = torch.device("cuda")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    idx = dv.build(up(cloud.positions), cam, cfg.pad)
    rays = (up(pixels), up(dirs), up(tn), up(tf), up(slopes))
    col = up(cloud.colors)
    for exact in (True, False):
        a = pipeline._query_sample(idx, col, *rays, hp.SamplerConfig(), exact, None, prefix=True)
        b = pipeline._query_sample(idx, col, *rays, hp.SamplerConfig(), exact, None, prefix=False)
        _assert_same(a.samples, b.samples)
        if want == 16:
            assert a.resorted > 0
        assert a.flagged <= a.resorted


def test_deferred_count_short_and_chunk_switch(monkeypatch):
    """The deferred head count (no host read between hp_head_count and the
    sampler): a remembered scratch size that is too small for this frame makes
    the sort write empty heads and the sampler's read raise CountShort; the
    frame re-runs reading the count and equals the full-CSR frame.  A frame
    that then needs ray chunks turns deferral off for the next frame (no
    wasted deferred pass), and a fitting frame turns it back on."""
    from paper_2404_14044_b200 import pipeline
    _, cloud, cam, cfg, tn, tf, stride, _ = gu.get_case("cfg1")
    dev = torch.device("cuda")
    xyz = torch.from_numpy(cloud.positions).to(dev)
    col = torch.from_numpy(cloud.colors).to(dev)
    pixels, dirs, t_near, t_far, slopes = gu.rays_and_slopes(cam, cfg, tn, tf, stride)
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rays = (up(pixels), up(dirs), up(t_near), up(t_far), up(slopes))
    idx = dv.build(xyz, cam, cfg.pad)
    sc = hp.SamplerConfig()
    full = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=False)
    dev = idx.device  # the library's per-device key (cuda:N)
    monkeypatch.setitem(dv._QUERY_CAP, dev, 1000)      # far below this frame's Q
    monkeypatch.setitem(dv._DEFER_OK, dev, True)
    calls = []
    orig = dv.CountShort.__init__
    monkeypatch.setattr(dv.CountShort, "__init__", lambda self, *a: (calls.append(a), orig(self, *a))[1])
    a = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=True)
    assert calls, "the deferred count should have run short"
    _assert_same(a.samples, full.samples)
    assert a.Q == full.Q
    # a smaller budget: the deferred attempt (the last frame fit) runs short,
    # the bound pass then shows the frame needs chunks
    b = pipeline._query_sample(idx, col, *rays, sc, True, max(full.Q // 5, 4096), prefix=True)
    assert b.chunks > 1 and dv._DEFER_OK[dev] is False and len(calls) == 2
    _assert_same(b.samples, full.samples)
    c = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=True)  # fits: read first, then defer again
    _assert_same(c.samples, full.samples)
    assert dv._DEFER_OK[dev] is True
    d = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=True)  # deferred, fits
    _assert_same(d.samples, full.samples)
    assert len(calls) == 2


def _dense_planes(stride=1):
    cloud = hp.generate_scene(hp.SceneSpec("parallel_planes", n=60_000, seed=3, plane_count=3,
                                           plane_gap=0.05, extent=0.8, noise=0.01))
    cam = hp.scene_camera(48, 40, fov_deg=14)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.04), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    dirs, pixels = dirs[::stride], pixels[::stride]
    tn, tf = np.full(len(dirs), 1.0), np.full(len(dirs), 10.0)
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
    dev = torch.device("cuda")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    idx = dv.build(up(cloud.positions), cam, cfg.pad)
    return cloud, idx, (up(pixels), up(dirs), up(tn), up(tf), up(slopes)), up(cloud.colors)


def test_long_head_resort_is_the_sorted_csr_head():
    """The long-head mode (hp_head_sort with whole up to 4096, re-sorting a
    subset from the same count pass): every head is the first plen entries
    of the full (t, id)-sorted CSR, up to ~4096 long."""
    _, idx, rays, _ = _dense_planes(stride=3)
    pre = dv.query_prefix(idx, *rays, want=16, whole=16)
    sel = torch.arange(0, int(rays[0].shape[0]), 2, device=rays[0].device)
    sub = dv.head_resort(pre, sel, want=dv.HEAD_LONG, whole=dv.HEAD_LONG)
    q = dv.query(idx, *[r[sel] for r in rays], facts=True)
    plen, counts = _check_prefix(q, sub, dv.HEAD_LONG)
    assert counts.max() > 1024 and plen.max() > 1024  # heads longer than the second chance's
    assert np.all(plen[counts <= dv.HEAD_LONG] == counts[counts <= dv.HEAD_LONG])


@pytest.mark.parametrize("gamma", [0.5, 0.3])
def test_pipeline_long_heads_equal_full(monkeypatch, gamma):
    """Rays whose exact transmittance needs more than 1024 candidates: the
    third chance (heads of up to 4096 from the same count pass) keeps them
    off the full query; the frame equals the full-CSR frame either way."""
    from paper_2404_14044_b200 import pipeline
    _, idx, rays, col = _dense_planes()
    sc = hp.SamplerConfig(gamma=gamma)
    b = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=False)
    flagged = {}
    for on, direct in ((False, 1.0), (True, 1.0), (True, 0.0)):  # direct 0: no 1024-entry second chance
        monkeypatch.setattr(pipeline, "LONG_HEADS", on)
        monkeypatch.setattr(pipeline, "LONG_DIRECT", direct)
        monkeypatch.setattr(pipeline, "LONG_BATCH", 97)  # several batches
        a = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=True)
        _assert_same(a.samples, b.samples)
        flagged[on, direct] = a.flagged
    assert flagged[False, 1.0] > 0 and flagged[True, 1.0] < flagged[False, 1.0]
    assert flagged[True, 0.0] == flagged[True, 1.0]


def test_pipeline_long_heads_after_1024_heads(monkeypatch):
    """Frames whose first heads are already 1024 long send flagged rays to
    the 4096-entry heads (not the full query); same frame as the full CSR."""
    from paper_2404_14044_b200 import pipeline
    monkeypatch.setattr(dv, "PREFIX_WANT", 1024)
    monkeypatch.setattr(dv, "HEAD_WHOLE", 1024)
    monkeypatch.setattr(pipeline, "LONG_DIRECT", 1.0)
    _, idx, rays, col = _dense_planes()
    sc = hp.SamplerConfig(gamma=0.5)
    b = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=False)
    a = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=True)
    _assert_same(a.samples, b.samples)
    assert a.resorted > 0 and a.flagged < a.resorted


@pytest.mark.parametrize("gamma", [0.9, 0.5])
def test_chunked_frame_long_first_equals_full(monkeypatch, gamma):
    """Ray chunks dense enough (footprint bound per ray over LONG_FIRST)
    start with the 4096-entry heads; the frame equals the full-CSR frame."""
    from paper_2404_14044_b200 import pipeline
    _, idx, rays, col = _dense_planes()
    sc = hp.SamplerConfig(gamma=gamma)
    b = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=False)
    for first in (1, 1 << 30):  # every chunk long-first / none
        monkeypatch.setattr(pipeline, "LONG_FIRST", first)
        a = pipeline._query_sample(idx, col, *rays, sc, True, max(b.Q // 4, 4096), prefix=True)
        assert a.chunks > 1
        _assert_same(a.samples, b.samples)
        assert a.Q == b.Q
