"""The reference's own hot-path tests, run against the B200 path.

Mirrors /root/reference/pkg/tests/test_hash_index.py (TestMortonCodes,
TestBuild, TestQuery, TestQueryBatch, TestInstrumentation) and
test_sampler.py (TestSampleRay, TestBatchSampler, TestGammaSweep) through this
package's drop-in API (numpy in / numpy out), with an independent numpy cone
oracle restated from the reference's tests/oracles.py:21-50.
"""

import os

import numpy as np
import pytest

import paper_2404_14044_b200 as hp
from paper_2404_14044_b200.hash_index import morton_codes, rasterize_points
from paper_2404_14044_b200.sampler import (confidence, make_candidates, pseudo_udf)

pytestmark = pytest.mark.gpu


def small_setup(n=2000, seed=0, width=32, height=24, scale=1.5, kind="uniform_box"):
    cloud = hp.generate_scene(hp.SceneSpec(kind=kind, n=n, seed=seed))
    camera = hp.scene_camera(width, height, fov_deg=45)
    return cloud, camera, hp.SearchConfig.for_camera(camera, scale=scale)


def cone_oracle(positions, ray, camera, config, restricted):
    """Vectorised cone query (independent of the package's kernels)."""
    if positions.shape[0] == 0:
        return np.empty(0, np.int64), np.empty(0), np.empty(0)
    px = positions - ray.origin
    t = px @ ray.direction
    dist = np.linalg.norm(px - t[:, None] * ray.direction, axis=1)
    slope = hp.radius_slope(camera, ray.pixel, config.kernel_radius, config.use_approx_radius)
    keep = (t >= ray.t_near) & (t <= ray.t_far) & (dist <= slope * t)
    if restricted:
        ok, pu, pv = rasterize_points(positions, camera, config.pad)
        cu, cv = ray.pixel[0] + config.pad, ray.pixel[1] + config.pad
        keep &= ok & (np.abs(pu - cu) <= config.pad) & (np.abs(pv - cv) <= config.pad)
    ids = np.flatnonzero(keep).astype(np.int64)
    order = np.lexsort((ids, t[ids]))
    return ids[order], t[ids][order], dist[ids][order]


def assert_result_equal(result, ids, ts, ds, atol=1e-12):
    np.testing.assert_array_equal(np.asarray(result.point_ids), ids)
    np.testing.assert_allclose(result.t_proj, ts, rtol=0, atol=atol)
    np.testing.assert_allclose(result.dist_perp, ds, rtol=0, atol=atol)


class TestBuild:
    def test_empty_cloud(self):
        cloud, camera, config = small_setup(n=0)
        index = hp.build(cloud, camera, config)
        assert index.reordered_ids.size == 0
        assert np.all(index.table_count == 0) and np.all(index.table_start == 0)

    def test_single_point_center_pixel(self):
        camera = hp.scene_camera(5, 5, fov_deg=40)
        cloud = hp.PointCloud((camera.origin + 3.0 * camera.forward).reshape(1, 3))
        index = hp.build(cloud, camera, hp.SearchConfig.for_camera(camera))
        assert index.table_count.sum() == 1
        lin = int(np.flatnonzero(index.table_count)[0])
        wp = index.padded_width
        assert (lin % wp - index.pad, lin // wp - index.pad) == (2, 2)

    def test_counts_match_projection_oracle(self):
        cloud, camera, config = small_setup(n=10000, seed=5)
        index = hp.build(cloud, camera, config)
        u, v, depth = camera.project(cloud.positions)
        pad = config.pad
        wp, hp_ = camera.width + 2 * pad, camera.height + 2 * pad
        fu, fv = np.floor(u) + pad, np.floor(v) + pad
        ok = (depth > 0) & (fu >= 0) & (fu < wp) & (fv >= 0) & (fv < hp_)
        expected = np.bincount((fv[ok] * wp + fu[ok]).astype(np.int64), minlength=wp * hp_)
        np.testing.assert_array_equal(index.table_count, expected)

    def test_points_behind_camera_dropped(self):
        camera = hp.scene_camera(8, 8)
        pts = np.array([[0, 0, 3.0], [0, 0, -3.0], [0.1, 0, 2.0]])
        index = hp.build(hp.PointCloud(pts), camera, hp.SearchConfig.for_camera(camera))
        assert index.indexed_count == 2
        assert 1 not in index.reordered_ids

    def test_ranges_contiguous_in_morton_order(self):
        cloud, camera, config = small_setup(n=5000, seed=2)
        index = hp.build(cloud, camera, config)
        wp, hp_ = index.padded_width, index.padded_height
        codes = morton_codes(np.tile(np.arange(wp, dtype=np.uint64), hp_),
                             np.repeat(np.arange(hp_, dtype=np.uint64), wp))
        occ = np.flatnonzero(index.table_count)
        by = occ[np.argsort(codes[occ])]
        np.testing.assert_array_equal(index.table_start[by],
                                      np.concatenate(([0], np.cumsum(index.table_count[by])[:-1])))

    def test_bijection_and_own_pixel_and_order(self):
        cloud, camera, config = small_setup(n=4000, seed=3)
        index = hp.build(cloud, camera, config)
        ok, pu, pv = rasterize_points(cloud.positions, camera, config.pad)
        np.testing.assert_array_equal(np.sort(index.reordered_ids), np.flatnonzero(ok))
        wp = index.padded_width
        for lin in np.flatnonzero(index.table_count)[::7]:
            s0, c = index.table_start[lin], index.table_count[lin]
            seg = index.reordered_ids[s0:s0 + c]
            assert np.all(pv[seg] * wp + pu[seg] == lin)
            assert np.all(np.diff(seg) > 0)

    def test_intra_pixel_order_ascending(self):
        camera = hp.scene_camera(4, 4)
        pts = np.tile(camera.origin + 3.0 * camera.forward, (5, 1))
        index = hp.build(hp.PointCloud(pts), camera, hp.SearchConfig.for_camera(camera))
        lin = int(np.flatnonzero(index.table_count)[0])
        s0, c = index.table_start[lin], index.table_count[lin]
        np.testing.assert_array_equal(index.reordered_ids[s0:s0 + c], np.arange(5))

    def test_many_points_in_one_pixel(self):
        """A bucket far above the small-bucket threshold (sorting network path)."""
        camera = hp.scene_camera(4, 4)
        rng = np.random.default_rng(0)
        pts = camera.origin + 3.0 * camera.forward + rng.uniform(-1e-6, 1e-6, (5000, 3))
        index = hp.build(hp.PointCloud(pts), camera, hp.SearchConfig.for_camera(camera))
        lin = int(np.argmax(index.table_count))
        s0, c = index.table_start[lin], index.table_count[lin]
        assert c > 1000
        assert np.all(np.diff(index.reordered_ids[s0:s0 + c]) > 0)

    def test_deterministic_and_touch_count(self):
        cloud, camera, config = small_setup(n=3000, seed=9)
        a, b = hp.build(cloud, camera, config), hp.build(cloud, camera, config)
        for k in ("table_start", "table_count", "reordered_ids", "slot_x"):
            np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
        assert a.point_touches == cloud.count + 2 * a.indexed_count

    def test_rejects_oversized_padded_image(self):
        camera = hp.scene_camera(70000, 4)
        with pytest.raises(ValueError, match="16-bit"):
            hp.build(hp.PointCloud(np.zeros((0, 3))), camera, hp.SearchConfig.for_camera(camera))


class TestQuery:
    def test_empty_index(self):
        cloud, camera, config = small_setup(n=0)
        index = hp.build(cloud, camera, config)
        assert len(hp.query(index, hp.generate_rays(camera, 1.0, 10.0)[0], config)) == 0

    def test_point_on_ray(self):
        cloud, camera, config = small_setup(n=0, width=9, height=9)
        ray = hp.generate_rays(camera, 1.0, 10.0)[4 * 9 + 4]
        t_mid = 0.5 * (ray.t_near + ray.t_far)
        index = hp.build(hp.PointCloud(ray.point_at(t_mid).reshape(1, 3)), camera, config)
        r = hp.query(index, ray, config)
        assert len(r) == 1 and r.point_ids[0] == 0
        assert r.t_proj[0] == pytest.approx(t_mid, abs=1e-12)
        assert r.dist_perp[0] == pytest.approx(0.0, abs=1e-12)

    @pytest.mark.parametrize("kind", ["uniform_box", "sphere_surface", "parallel_planes"])
    def test_matches_restricted_oracle(self, kind):
        cloud, camera, config = small_setup(n=5000, seed=11, kind=kind)
        index = hp.build(cloud, camera, config)
        rays = hp.generate_rays(camera, 1.0, 10.0)
        sel = np.random.default_rng(0).choice(len(rays), size=300, replace=False)
        res = hp.query_batch(index, [rays[i] for i in sel], config)
        total = 0
        for r, i in zip(res, sel):
            assert_result_equal(r, *cone_oracle(cloud.positions, rays[i], camera, config, True))
            total += len(r)
        assert total > 0

    def test_result_invariants(self):
        cloud, camera, config = small_setup(n=5000, seed=13)
        index = hp.build(cloud, camera, config)
        rays = hp.generate_rays(camera, 1.0, 10.0)[100:200]
        for ray, r in zip(rays, hp.query_batch(index, rays, config)):
            slope = hp.radius_slope(camera, ray.pixel, config.kernel_radius)
            assert np.all(np.diff(r.t_proj) >= 0)
            assert np.unique(r.point_ids).size == len(r)
            assert np.all((r.t_proj >= ray.t_near) & (r.t_proj <= ray.t_far))
            assert np.all(r.dist_perp <= slope * r.t_proj + 1e-15)

    def test_padding_keeps_border_points_findable(self):
        camera = hp.scene_camera(16, 16, fov_deg=40)
        config = hp.SearchConfig.for_camera(camera, scale=2.0)
        ray = hp.generate_rays(camera, 1.0, 10.0)[0]
        base = ray.point_at(4.0)
        off = camera.pixel_width * 4.0 * 1.2
        pts = np.array([base - off * camera.right, base - off * camera.right + 0.001 * camera.up])
        index = hp.build(hp.PointCloud(pts), camera, config)
        assert index.indexed_count == 2
        assert_result_equal(hp.query(index, ray, config), *cone_oracle(pts, ray, camera, config, True))

    def test_rejects_foreign_pixel_origin_kernel(self):
        cloud, camera, config = small_setup(n=10, scale=1.5)
        index = hp.build(cloud, camera, config)
        with pytest.raises(ValueError, match="pixel"):
            hp.query(index, hp.Ray(camera.origin, camera.forward, 1.0, 10.0, (camera.width, 0)), config)
        with pytest.raises(ValueError, match="origin"):
            hp.query(index, hp.Ray(camera.origin + [0, 0, 0.5], camera.forward, 1.0, 10.0, (0, 0)),
                     config)
        other = hp.SearchConfig.for_camera(camera, scale=3.5)
        with pytest.raises(ValueError, match="kernel size"):
            hp.query(index, hp.generate_rays(camera, 1.0, 10.0)[0], other)


class TestQueryBatch:
    def test_batch_of_one_and_permutation(self):
        cloud, camera, config = small_setup(n=1500, seed=22)
        index = hp.build(cloud, camera, config)
        rays = hp.generate_rays(camera, 1.0, 10.0)[50:80]
        single = hp.query(index, rays[7], config)
        [batched] = hp.query_batch(index, [rays[7]], config)
        np.testing.assert_array_equal(batched.point_ids, single.point_ids)
        perm = np.random.default_rng(0).permutation(len(rays))
        out = hp.query_batch(index, rays, config)
        out_p = hp.query_batch(index, [rays[i] for i in perm], config)
        for j, i in enumerate(perm):
            np.testing.assert_array_equal(out_p[j].point_ids, out[i].point_ids)
            np.testing.assert_array_equal(out_p[j].t_proj, out[i].t_proj)

    def test_full_frame_equals_sequential_and_parallel(self, monkeypatch):
        cloud, camera, config = small_setup(n=2500, seed=23, kind="parallel_planes")
        index = hp.build(cloud, camera, config)
        rays = hp.generate_rays(camera, 1.0, 10.0)
        batch = hp.query_batch(index, rays, config)
        monkeypatch.setenv("HASHPOINT_THREADS", "3")
        par = hp.query_batch(index, rays, config, parallel=True)
        for i in range(0, len(rays), 37):
            single = hp.query(index, rays[i], config)
            for r in (batch[i], par[i]):
                np.testing.assert_array_equal(r.point_ids, single.point_ids)
                np.testing.assert_array_equal(r.t_proj, single.t_proj)
                np.testing.assert_array_equal(r.dist_perp, single.dist_perp)


class TestInstrumentation:
    def test_probe_and_scan_counts(self):
        cloud, camera, config = small_setup(n=3000, seed=31)
        index = hp.build(cloud, camera, config)
        dirs, pixels = hp.ray_grid(camera)
        m = len(dirs)
        _, _, _, _, probes, scanned = hp.query_batch_arrays(index, pixels, dirs, np.full(m, 1.0),
                                                            np.full(m, 10.0), config)
        s = config.kernel_size
        assert np.all(probes == s * s)
        wp, pad = index.padded_width, index.pad
        for i in range(0, m, 53):
            cu, cv = pixels[i] + pad
            expect = sum(index.table_count[(cv + dv) * wp + cu + du]
                         for dv in range(-pad, pad + 1) for du in range(-pad, pad + 1))
            assert scanned[i] == expect


def planes_setup(gap=1.5, n=6000, count=2, width=24, height=24, noise=0.0, extent=2.0):
    cloud = hp.generate_scene(hp.SceneSpec(kind="parallel_planes", n=n, seed=0, plane_count=count,
                                           plane_gap=gap, noise=noise, extent=extent))
    camera = hp.scene_camera(width, height, fov_deg=30)
    config = hp.SearchConfig.for_camera(camera, scale=2.0)
    return cloud, camera, config, hp.build(cloud, camera, config), hp.generate_rays(camera, 1.0, 10.0)


class TestSampler:
    def test_empty_scene(self):
        cloud, camera, config, index, rays = planes_setup(n=0)
        assert hp.sample_ray(index, rays[0]) == []

    def test_dense_plane_samples_near_surface(self):
        cloud, camera, config, index, rays = planes_setup(count=1, n=8000)
        cfg = hp.SamplerConfig()
        hit = 0
        for ray in rays[len(rays) // 2 - 12: len(rays) // 2 + 12]:
            kept = hp.sample_ray(index, ray, config, cfg)
            hit += bool(kept)
            for c in kept:
                assert abs(c.position[2] - 4.0) <= 3 * cfg.beta
        assert hit > 0

    def test_six_surfaces_primary_dominates(self):
        cloud, camera, config, index, rays = planes_setup(count=6, gap=1.0, n=30000, extent=1.0)
        cfg = hp.SamplerConfig(gamma=0.9, epsilon=1e-4)
        checked = 0
        for ray in rays[len(rays) // 2 - 20: len(rays) // 2 + 20]:
            kept = hp.sample_ray(index, ray, config, cfg)
            checked += bool(kept)
            for c in kept:
                assert abs(c.position[2] - 1.5) <= 3 * cfg.beta
        assert checked > 10

    @pytest.mark.parametrize("mode", ["epsilon", "tau"])
    def test_batch_equals_scalar_pipeline(self, mode):
        cloud, camera, config, index, rays = planes_setup(n=4000, noise=0.05)
        cfg = hp.SamplerConfig(retention_mode=mode)
        subset = rays[::7]
        pixels = np.array([r.pixel for r in subset], np.int64)
        dirs = np.array([r.direction for r in subset])
        tn, tf = np.full(len(subset), 1.0), np.full(len(subset), 10.0)
        off, ids, t, dist, _, _ = hp.query_batch_arrays(index, pixels, dirs, tn, tf, config)
        slopes = hp.radius_slopes(camera, pixels, config.kernel_radius)
        roff, rid, rt, _, rudf, ralpha, rw, _, _ = hp.sample_batch_arrays(off, ids, t, dist, slopes, cfg)
        for i, ray in enumerate(subset):
            res = hp.query(index, ray, config)
            cands = make_candidates(res, ray, camera, config)
            for c in cands:
                c.udf_distance = pseudo_udf(c, res, cfg.k_neighbors)
                c.confidence = confidence(c.udf_distance, cfg.beta, cfg.gamma)
            hp.occlusion_weights(cands)
            kept = hp.retain(cands, cfg)
            lo, hi = roff[i], roff[i + 1]
            assert hi - lo == len(kept)
            np.testing.assert_array_equal(rid[lo:hi], [c.point_id for c in kept])
            np.testing.assert_allclose(rudf[lo:hi], [c.udf_distance for c in kept], rtol=1e-9)
            np.testing.assert_allclose(ralpha[lo:hi], [c.confidence for c in kept], rtol=1e-9)
            np.testing.assert_allclose(rw[lo:hi], [c.weight for c in kept], rtol=1e-9, atol=1e-15)

    def test_transmittance_covers_all_candidates(self):
        cloud, camera, config, index, rays = planes_setup(n=4000)
        cfg = hp.SamplerConfig()
        subset = rays[::11]
        pixels = np.array([r.pixel for r in subset], np.int64)
        dirs = np.array([r.direction for r in subset])
        m = len(subset)
        off, ids, t, dist, _, _ = hp.query_batch_arrays(index, pixels, dirs, np.full(m, 1.0),
                                                        np.full(m, 10.0), config)
        slopes = hp.radius_slopes(camera, pixels, config.kernel_radius)
        t_end = hp.sample_batch_arrays(off, ids, t, dist, slopes, cfg)[8]
        for i, ray in enumerate(subset):
            res = hp.query(index, ray, config)
            cands = make_candidates(res, ray, camera, config)
            alphas = [confidence(pseudo_udf(c, res, cfg.k_neighbors), cfg.beta, cfg.gamma)
                      for c in cands]
            expected = np.prod([1.0 - a for a in alphas]) if cands else 1.0
            assert t_end[i] == pytest.approx(expected, rel=1e-9, abs=1e-300)

    def test_gamma_sweep_monotone(self):
        cloud, camera, config, index, rays = planes_setup(count=2, gap=1.5, n=8000)
        subset = rays[::5]
        counts = np.array([[len(hp.sample_ray(index, r, config, hp.SamplerConfig(gamma=g)))
                            for r in subset] for g in (0.1, 0.3, 0.5, 0.7, 0.9)])
        assert np.all(np.diff(counts, axis=0) <= 0)
        assert counts[0].sum() > counts[-1].sum()

    def test_unsorted_input_uses_reference_loops(self):
        """sample_batch_arrays accepts any CSR; unsorted t takes the direct path."""
        from oracle import oracle as orc
        rng = np.random.default_rng(3)
        q = 40
        off = np.array([0, q, q, 2 * q], np.int64)
        ids = np.arange(2 * q, dtype=np.int64)
        t = rng.uniform(1, 2, 2 * q)
        d = rng.uniform(0, 0.05, 2 * q)
        slopes = np.array([0.03, 0.03, 0.03])
        cfg = hp.SamplerConfig(gamma=0.4, epsilon=1e-3)
        got = hp.sample_batch_arrays(off, ids, t, d, slopes, cfg)
        ref = orc.sample(off, ids, t, d, slopes, cfg.k_neighbors, cfg.beta ** 2, cfg.gamma, True,
                         cfg.epsilon, cfg.tau_min)
        for a, b in zip(got[:5], ref[:5]):
            np.testing.assert_array_equal(a, b)
        for a, b in zip(got[5:], ref[5:]):
            np.testing.assert_allclose(a, b, rtol=1e-12)
