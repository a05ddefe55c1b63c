"""Long query segments: rays whose match count q falls in the 4096-class and
the global-memory class of the sort (q > 4096), and the large-K sampler
(K > 32: the dynamic K-best list), against the C oracle bit for bit.

Reference behaviour: _kernels.hash_query_batch (_kernels.py:86-157) and
_kernels.sample_batch (_kernels.py:552-700) have no size limits; the device
path switches algorithms by size, so every class is checked here.
"""

import numpy as np
import pytest
import torch

import paper_2404_14044_b200 as hp
from oracle import oracle as orc
from paper_2404_14044_b200 import device as dv

pytestmark = pytest.mark.gpu


def _oracle_query(cloud, cam, cfg, pixels, dirs, tn, tf, slopes):
    ob = orc.build(cloud.positions, cam, cfg.pad)
    return orc.query(ob["table_start"], ob["table_count"], ob["slot_x"], ob["slot_y"], ob["slot_z"],
                     ob["reordered_ids"], cam.width + 2 * cfg.pad, cfg.pad, pixels[:, 0], pixels[:, 1],
                     dirs, cam.origin, tn, tf, slopes, threads=8)


@pytest.fixture(scope="module")
def dense_case():
    # a dense, noisy slab right in front of a narrow camera, wide cones:
    # q from a few hundred to ~7700 matches per ray
    cloud = hp.generate_scene(hp.SceneSpec("parallel_planes", n=60_000, seed=3, plane_count=3,
                                           plane_gap=0.05, extent=0.8, noise=0.01))
    cam = hp.scene_camera(48, 40, fov_deg=14)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.04), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    sel = np.arange(0, dirs.shape[0], 29)
    m = sel.size
    tn, tf = np.full(m, 1.0), np.full(m, 10.0)
    slopes = hp.radius_slopes(cam, pixels[sel], cfg.kernel_radius)
    c = np.diff(_oracle_query(cloud, cam, cfg, pixels[sel], dirs[sel], tn, tf, slopes)[0])
    # keep every class but only a few of the (oracle-expensive) longest rays
    keep = np.concatenate([np.flatnonzero(c > 4096)[:6], np.flatnonzero(c <= 4096)])
    sel = np.sort(sel[keep])
    dirs, pixels = dirs[sel], pixels[sel]
    m = sel.size
    tn, tf = np.full(m, 1.0), np.full(m, 10.0)
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
    oq = _oracle_query(cloud, cam, cfg, pixels, dirs, tn, tf, slopes)
    dev = torch.device("cuda")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    idx = dv.build(up(cloud.positions), cam, cfg.pad)
    q = dv.query(idx, up(pixels), up(dirs), up(tn), up(tf), up(slopes))
    return cloud, q, oq, up(slopes), slopes


def test_dense_query_covers_every_sort_class_and_is_bit_exact(dense_case):
    cloud, q, oq, _, _ = dense_case
    counts = np.diff(oq[0])
    assert (counts > 4096).sum() >= 3, counts.max()           # 8192 class
    assert ((counts > 2048) & (counts <= 4096)).sum() >= 3     # 4096 class
    assert ((counts > 1024) & (counts <= 2048)).sum() >= 3     # 2048 class
    for a, b in zip(q, oq):
        np.testing.assert_array_equal(a.cpu().numpy(), b)


@pytest.mark.parametrize("k,mode,gamma", [(8, "epsilon", 0.9), (40, "epsilon", 0.5), (3, "tau", 0.3)])
@pytest.mark.parametrize("exact_t_end", [True, False])
def test_dense_sampling_matches_oracle(dense_case, k, mode, gamma, exact_t_end):
    cloud, q, oq, slopes_d, slopes = dense_case
    sc = hp.SamplerConfig(k_neighbors=k, retention_mode=mode, gamma=gamma)
    col = torch.from_numpy(cloud.colors).cuda()
    out = [x.cpu().numpy() for x in dv.sample(q[0], q[1], q[2], q[3], slopes_d, sc, col,
                                               exact_t_end=exact_t_end)]
    ref = orc.sample(oq[0], oq[1], oq[2], oq[3], slopes, k, sc.beta * sc.beta, gamma, mode == "epsilon",
                     sc.epsilon, sc.tau_min, cloud.colors, threads=8)
    for i in range(5):  # offsets, ids, t, dist, udf: bit-exact
        np.testing.assert_array_equal(out[i], ref[i])
    for i in (5, 6, 7):  # alpha, w, colour: device exp vs glibc exp
        np.testing.assert_allclose(out[i], ref[i], rtol=1e-12, atol=1e-300)
    if exact_t_end:
        np.testing.assert_allclose(out[8], ref[8], rtol=1e-12, atol=1e-300)


def test_huge_rays_split_into_parts_bit_exact():
    """q up to ~32k: rays above the largest shared-memory class are split into
    t-ordered parts sorted in place; the CSR and (for a few rays) the samples
    match the oracle bit for bit."""
    cloud = hp.generate_scene(hp.SceneSpec("parallel_planes", n=200_000, seed=3, plane_count=3,
                                           plane_gap=0.05, extent=0.8, noise=0.01))
    cam = hp.scene_camera(48, 40, fov_deg=14)
    cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.045), hp.pixel_disc_radius(cam))
    dirs, pixels = hp.ray_grid(cam)
    sel = np.arange(0, dirs.shape[0], 37)
    dirs, pixels = dirs[sel], pixels[sel]
    m = sel.size
    tn, tf = np.full(m, 1.0), np.full(m, 10.0)
    slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
    oq = _oracle_query(cloud, cam, cfg, pixels, dirs, tn, tf, slopes)
    counts = np.diff(oq[0])
    assert (counts > 16384).sum() >= 3, counts.max()
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    idx = dv.build(up(cloud.positions), cam, cfg.pad)
    q = dv.query(idx, up(pixels), up(dirs), up(tn), up(tf), up(slopes))
    for a, b in zip(q, oq):
        np.testing.assert_array_equal(a.cpu().numpy(), b)
    # samples of three of the longest rays
    pick = np.argsort(-counts)[:3]
    sub = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    rows = []
    for r in pick:
        a, b = oq[0][r], oq[0][r + 1]
        rows.append((a, b))
    off = np.concatenate([[0], np.cumsum([b - a for a, b in rows])])
    cat = lambda arr: np.concatenate([arr[a:b] for a, b in rows])  # noqa: E731
    ids, t, d, sl = cat(oq[1]), cat(oq[2]), cat(oq[3]), slopes[pick]
    sc = hp.SamplerConfig()
    out = [x.cpu().numpy() for x in dv.sample(sub(off), sub(ids), sub(t), sub(d), sub(sl), sc,
                                               torch.from_numpy(cloud.colors).cuda())]
    ref = orc.sample(off, ids, t, d, sl, sc.k_neighbors, sc.beta * sc.beta, sc.gamma, True, sc.epsilon,
                     sc.tau_min, cloud.colors, threads=3)
    for i in range(5):
        np.testing.assert_array_equal(out[i], ref[i])
    for i in (5, 6, 7, 8):
        np.testing.assert_allclose(out[i], ref[i], rtol=1e-12, atol=1e-300)
