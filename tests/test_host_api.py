"""Host-side logic of the drop-in (CPU only): types, validation, error
messages, utilities, and the scalar sampler helpers — mirroring the
reference's own unit tests (test_geometry.py, test_hash_index.py,
test_sampler.py) where they do not need the device."""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2404_14044_b200 as hp
from paper_2404_14044_b200.hash_index import morton_codes
from paper_2404_14044_b200.sampler import (SampleCandidate, confidence, occlusion_weights,
                                           pseudo_udf, retain)


class TestMorton:
    def test_known_values(self):  # reference test_hash_index.py:33-38
        u = np.array([0, 1, 2, 3, 3], np.uint64)
        v = np.array([0, 0, 1, 5, 3], np.uint64)
        np.testing.assert_array_equal(morton_codes(u, v), [0, 1, 6, 39, 15])

    def test_unique_on_grid(self):
        w, h = 37, 23
        codes = morton_codes(np.tile(np.arange(w, dtype=np.uint64), h),
                             np.repeat(np.arange(h, dtype=np.uint64), w))
        assert np.unique(codes).size == w * h

    @pytest.mark.parametrize("wp,hp", [(1, 1), (5, 3), (37, 23), (840, 840), (1, 300), (300, 2)])
    def test_device_rank_formula_matches_sorted_codes(self, wp, hp):
        """The quadtree rank used by k_morton_permute (hp_build.cu) equals the
        position of each pixel in the stable argsort of Morton codes."""
        levels = 0
        while (1 << levels) < max(wp, hp):
            levels += 1

        def rank(u, v):
            r, bu, bv = 0, 0, 0
            for lv in range(levels - 1, -1, -1):
                h = 1 << lv
                q = ((u >> lv) & 1) | (((v >> lv) & 1) << 1)
                for k in range(q):
                    x0, y0 = bu + (k & 1) * h, bv + (k >> 1) * h
                    w_ = (min(x0 + h, wp) - x0) if x0 < wp else 0
                    h_ = (min(y0 + h, hp) - y0) if y0 < hp else 0
                    r += w_ * h_
                bu += (q & 1) * h
                bv += (q >> 1) * h
            return r

        gu = np.tile(np.arange(wp, dtype=np.uint64), hp)
        gv = np.repeat(np.arange(hp, dtype=np.uint64), wp)
        order = np.argsort(morton_codes(gu, gv), kind="stable")
        expect = np.empty(wp * hp, np.int64)
        expect[order] = np.arange(wp * hp)
        rng = np.random.default_rng(0)
        sel = rng.choice(wp * hp, size=min(wp * hp, 2000), replace=False)
        got = np.array([rank(int(l % wp), int(l // wp)) for l in sel])
        np.testing.assert_array_equal(got, expect[sel])


class TestGeometry:
    def test_disc_radius_and_kernel_size(self):
        cam = hp.Camera(np.zeros(3), np.eye(3), 1.0, 4, 4, math.sqrt(math.pi), math.sqrt(math.pi))
        assert hp.pixel_disc_radius(cam) == pytest.approx(1.0)
        assert hp.kernel_size(0.0, 1.0) == 1
        assert hp.kernel_size(1.0, 1.0) == 3
        assert hp.kernel_size(1.01, 1.0) == 5

    def test_cfg2_kernel(self):
        cam = hp.scene_camera(800, 800, fov_deg=40)
        cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.01),
                              hp.pixel_disc_radius(cam))
        assert (cfg.kernel_size, cfg.pad) == (41, 20)

    def test_camera_validation(self):
        with pytest.raises(ValueError, match="orthonormal"):
            hp.Camera(np.zeros(3), np.ones((3, 3)), 1.0, 4, 4, 0.1, 0.1)
        with pytest.raises(ValueError, match="positive"):
            hp.Camera(np.zeros(3), np.eye(3), 0.0, 4, 4, 0.1, 0.1)
        with pytest.raises(ValueError, match="1x1"):
            hp.Camera(np.zeros(3), np.eye(3), 1.0, 0, 4, 0.1, 0.1)
        with pytest.raises(ValueError, match="colinear"):
            hp.Camera.from_vectors(np.zeros(3), [0, 1, 0], [0, 1, 0], 1.0, 4, 4, 0.1, 0.1)

    def test_ray_validation(self):
        with pytest.raises(ValueError, match="unit"):
            hp.Ray(np.zeros(3), [0, 0, 2.0], 1.0, 2.0, (0, 0))
        with pytest.raises(ValueError, match="t_near"):
            hp.Ray(np.zeros(3), [0, 0, 1.0], 2.0, 1.0, (0, 0))

    def test_search_config_validation(self):
        with pytest.raises(ValueError):
            hp.SearchConfig(1.0, 0.0)
        with pytest.raises(ValueError):
            hp.SearchConfig(-1.0, 1.0)

    def test_ray_grid_row_major_unit(self):
        cam = hp.scene_camera(7, 5)
        dirs, pix = hp.ray_grid(cam)
        assert dirs.shape == (35, 3) and pix.shape == (35, 2)
        np.testing.assert_array_equal(pix[8], [1, 1])
        np.testing.assert_allclose(np.linalg.norm(dirs, axis=1), 1.0, atol=1e-15)

    def test_scalar_and_vector_slopes_agree(self):
        cam = hp.scene_camera(40, 30)
        _, pix = hp.ray_grid(cam)
        for approx in (False, True):
            vec = hp.radius_slopes(cam, pix, 0.01, approx)
            sca = [hp.radius_slope(cam, tuple(p), 0.01, approx) for p in pix[::37]]
            np.testing.assert_allclose(vec[::37], sca, rtol=1e-15)


class TestQueryResult:
    def test_roundtrip(self):
        out = hp.results_from_csr(np.array([0, 2, 2, 3]), np.array([5, 7, 9]),
                                  np.array([1.0, 2.0, 3.0]), np.array([0.1, 0.2, 0.3]))
        assert [len(r) for r in out] == [2, 0, 1]
        assert out[2].point_ids[0] == 9

    def test_validates(self):
        with pytest.raises(ValueError):
            hp.QueryResult(np.array([1]), np.array([1.0, 2.0]), np.array([0.0]))


class TestSamplerHost:
    def test_defaults(self):
        cfg = hp.SamplerConfig()
        assert (cfg.k_neighbors, cfg.gamma, cfg.retention_mode) == (8, 0.9, "epsilon")
        assert cfg.beta ** 2 == pytest.approx(0.02)

    @pytest.mark.parametrize("kw", [dict(k_neighbors=0), dict(beta=0.0), dict(gamma=0.0),
                                    dict(gamma=1.5), dict(retention_mode="x"),
                                    dict(epsilon=-1.0), dict(tau_min=1.0)])
    def test_validation(self, kw):
        with pytest.raises(ValueError):
            hp.SamplerConfig(**kw)

    @staticmethod
    def _res(ts, ds):
        return hp.QueryResult(np.arange(len(ts)), np.asarray(ts, float), np.asarray(ds, float))

    @staticmethod
    def _cand(t, radius=1.0):
        return SampleCandidate(t=t, position=np.zeros(3), radius=radius, dist_perp=0.0, point_id=0)

    def test_pseudo_udf_kats(self):  # reference test_sampler.py:98-140
        assert pseudo_udf(self._cand(2.0, 0.5), self._res([2.0] * 3, [0.0] * 3), 3) == 0.0
        assert pseudo_udf(self._cand(2.0), self._res([2.0], [0.3]), 1) == pytest.approx(0.3)
        got = pseudo_udf(self._cand(2.0, 0.1), self._res([2.0, 2.0, 2.001, 2.001],
                                                          [0.05, 0.06, 0.2, 0.21]), 2)
        assert got == pytest.approx(0.055, rel=1e-12)
        got = pseudo_udf(self._cand(2.0, 0.1), self._res([2.0, 2.0, 2.0], [0.05, 0.2, 0.3]), 2)
        assert got == pytest.approx(0.125, rel=1e-12)
        got = pseudo_udf(self._cand(2.0, 5.0), self._res([2.0, 2.5], [0.1, 0.1]), 8)
        assert got == pytest.approx(np.mean([0.1, np.hypot(0.5, 0.1)]), rel=1e-12)
        with pytest.raises(ValueError):
            pseudo_udf(self._cand(1.0), hp.QueryResult.empty(), 4)

    def test_confidence(self):
        assert confidence(0.0, 0.5, 0.8) == 0.8
        assert confidence(0.7, 0.7, 1.0) == pytest.approx(math.exp(-1), rel=1e-15)
        with pytest.raises(ValueError):
            confidence(-1.0, 1.0, 0.5)

    @given(d1=st.floats(0, 3), delta=st.floats(1e-6, 3))
    @settings(deadline=None, max_examples=50)
    def test_confidence_decreasing(self, d1, delta):
        a1, a2 = confidence(d1, 0.5, 0.9), confidence(d1 + delta, 0.5, 0.9)
        assert a1 > a2 or a2 == 0.0

    def _weighted(self, alphas):
        cands = [self._cand(float(k + 1)) for k in range(len(alphas))]
        for c, a in zip(cands, alphas):
            c.confidence = a
        return occlusion_weights(cands)

    def test_weights_and_retention(self):  # reference test_sampler.py:182-263
        assert [c.weight for c in self._weighted([0.5, 0.5])] == [0.5, 0.25]
        assert [c.weight for c in self._weighted([1.0, 0.7])] == [1.0, 0.0]
        kept = retain(self._weighted([0.9, 0.9, 0.9, 0.9]),
                      hp.SamplerConfig(retention_mode="tau", tau_min=0.05))
        assert len(kept) == 2
        assert len(retain(self._weighted([1e-8, 0.9]),
                          hp.SamplerConfig(retention_mode="tau", tau_min=0.01))) == 2
        with pytest.raises(ValueError, match="sorted"):
            cs = [self._cand(2.0), self._cand(1.0)]
            for c in cs:
                c.confidence = 0.5
            occlusion_weights(cs)

    def test_primary_surface_host(self):
        pid, pt = hp.primary_surface(np.array([0, 2, 2, 3]), np.array([7, 8, 9]),
                                     np.array([1.5, 2.5, 3.5]))
        np.testing.assert_array_equal(pid, [7, -1, 9])
        assert pt[0] == 1.5 and np.isnan(pt[1]) and pt[2] == 3.5


class TestScenes:
    def test_deterministic_and_shaped(self):
        a = hp.generate_scene(hp.SceneSpec("parallel_planes", n=1001, seed=4, plane_count=3))
        b = hp.generate_scene(hp.SceneSpec("parallel_planes", n=1001, seed=4, plane_count=3))
        np.testing.assert_array_equal(a.positions, b.positions)
        assert a.positions.shape == (1001, 3) and a.colors.shape == (1001, 3)

    def test_validation(self):
        with pytest.raises(ValueError):
            hp.SceneSpec("nope")
        with pytest.raises(ValueError):
            hp.SceneSpec("uniform_box", n=-1)


def test_native_host_slopes_are_bit_identical():
    import paper_2404_14044_b200 as hp
    from paper_2404_14044_b200 import pipeline
    from paper_2404_14044_b200.geometry import radius_slopes
    cam = hp.scene_camera(320, 240, fov_deg=60, origin=(0.3, -0.2, 0.1), target=(0.0, 0.1, 4.0))
    dirs, pix = hp.ray_grid(cam)
    for approx in (False, True):
        a = radius_slopes(cam, pix, 0.0137, approx)
        for threads in (1, 7):
            b = pipeline.host_slopes(cam, pix, 0.0137, approx, threads=threads)
            assert a.tobytes() == b.tobytes()
            g = pipeline.host_slopes(cam, None, 0.0137, approx, threads=threads)  # the ray grid
            assert a.tobytes() == g.tobytes()
