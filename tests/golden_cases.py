"""Definitions of the golden parity cases.

Shared by ``oracle/make_golden.py`` (which runs the REFERENCE package on these
inputs, in the dev container only) and the tests (which rebuild the same inputs
with this package's own seeded generators and compare the oracle / the device
path against the stored outputs).  Inputs are regenerated, never stored: the
fixture records a sha256 of the generated positions to prove both sides saw
the same cloud.
"""

from __future__ import annotations

import numpy as np

from paper_2404_14044_b200.cloud import PointCloud
from paper_2404_14044_b200.geometry import (SearchConfig, kernel_radius_for_min_radius,
                                            ray_grid)
from paper_2404_14044_b200.scenes import SceneSpec, generate_scene, scene_camera

# sampler configurations (k, beta, gamma, mode, eps, tau) exercised per case
SAMPLERS = {
    "default": dict(),
    "tau": dict(retention_mode="tau", tau_min=0.01),
    "k3_g05": dict(k_neighbors=3, gamma=0.5),
    "k1": dict(k_neighbors=1),
    "k20_g01": dict(k_neighbors=20, gamma=0.1, epsilon=1e-3),
    "tau_g03": dict(retention_mode="tau", gamma=0.3, tau_min=0.2),
}


def _orbit_camera(width, height, k, count=64, fov=60.0):
    th = 2.0 * np.pi * k / count
    return scene_camera(width, height, fov_deg=fov,
                        origin=(0.4 * np.cos(th), 0.4 * np.sin(th), 0.0), target=(0.0, 0.0, 4.0))


def _dup_planes():
    base = generate_scene(SceneSpec("parallel_planes", n=3000, seed=5, plane_count=2,
                                    plane_gap=0.7, noise=0.0, extent=1.5))
    pos = np.repeat(base.positions, 3, axis=0)                       # exact d^2 ties
    rgb = np.tile(np.array([[0.1, 0.2, 0.3], [0.9, 0.5, 0.1], [0.4, 0.4, 0.8]]),
                  (base.count, 1))
    return PointCloud(pos, rgb)


def _edge_points(camera):
    o, f = camera.origin, camera.forward
    pts = [o + 3.0 * f, o + 3.0 * f, o + 3.0 * f,                   # coincident (ties)
           o - 3.0 * f,                                              # behind camera
           o + 2.0 * f + 0.001 * camera.right,
           o + 9.99 * f, o + 10.5 * f, o + 0.5 * f]                   # t bounds
    # just outside the image, inside the padded margin
    pts.append(camera.pixel_center(0, 0) * 4.0 - 4.0 * 1.2 * camera.pixel_width * camera.right)
    return PointCloud(np.array(pts), np.full((len(pts), 3), 0.5))


def cases():
    """Yield (name, cloud, camera, search_config, t_near, t_far, ray_stride, samplers)."""
    # cfg1 of BASELINE.json: 100k sphere shell, 200x200, delta = 0.01
    cam = scene_camera(200, 200, fov_deg=40)
    cfg = SearchConfig(kernel_radius_for_min_radius(cam, 1.0, 0.01),
                       SearchConfig.for_camera(cam).pixel_disc_radius)
    yield ("cfg1", generate_scene(SceneSpec("sphere_surface", n=100_000, seed=0, noise=0.005)),
           cam, cfg, 1.0, 10.0, 1, ["default", "tau"])
    for kind, seed in (("uniform_box", 11), ("sphere_surface", 12), ("parallel_planes", 13)):
        cam = scene_camera(32, 24, fov_deg=45)
        yield (f"small_{kind}", generate_scene(SceneSpec(kind, n=5000, seed=seed, noise=0.01)),
               cam, SearchConfig.for_camera(cam, scale=1.5), 1.0, 10.0, 1,
               ["default", "tau", "k3_g05", "k1"])
    # rotated, off-origin camera (projection op-order sensitivity), approx radius
    cam = _orbit_camera(64, 48, 5)
    yield ("orbit_planes", generate_scene(SceneSpec("parallel_planes", n=30_000, seed=3,
                                                    plane_count=6, plane_gap=0.5, extent=4.0,
                                                    noise=0.005)),
           cam, SearchConfig.for_camera(cam, scale=3.0, use_approx_radius=True), 1.0, 10.0, 1,
           ["default", "tau", "k20_g01"])
    cam = scene_camera(24, 24, fov_deg=30)
    yield ("dup_planes", _dup_planes(), cam, SearchConfig.for_camera(cam, scale=2.0), 1.0, 10.0,
           1, ["default", "tau", "k3_g05", "tau_g03"])
    cam = scene_camera(9, 9, fov_deg=40)
    yield ("edge_points", _edge_points(cam), cam, SearchConfig.for_camera(cam, scale=2.0),
           1.0, 10.0, 1, ["default", "tau", "k1"])
    cam = scene_camera(16, 12, fov_deg=40)
    yield ("empty", PointCloud(np.zeros((0, 3)), np.zeros((0, 3))), cam,
           SearchConfig.for_camera(cam), 1.0, 10.0, 1, ["default"])


def rays_for(camera, t_near, t_far, stride=1):
    dirs, pixels = ray_grid(camera)
    dirs, pixels = dirs[::stride], pixels[::stride]
    m = dirs.shape[0]
    return pixels, dirs, np.full(m, t_near), np.full(m, t_far)


# render configurations: (tag, mode, background, knp_k, sampler)
RENDERS = [
    ("vol", "volume", (0.0, 0.0, 0.0), 8, "default"),
    ("vol_bg_tau", "volume", (0.2, 0.5, 1.0), 8, "tau"),
    ("knp", "knp_blend", (0.0, 0.0, 0.0), 8, "default"),
    ("knp3_bg", "knp_blend", (0.1, 0.1, 0.1), 3, "k3_g05"),
    ("knp1", "knp_blend", (1.0, 1.0, 1.0), 1, "default"),
]


def render_cases():
    """Yield (name, cloud, camera, search_config, t_near, t_far, render configs) for the
    renderer goldens (reference renderer.py:138-192 over generate_rays)."""
    byname = {c[0]: c for c in cases()}
    for name in ("small_sphere_surface", "orbit_planes", "dup_planes", "edge_points"):
        _, cloud, cam, cfg, tn, tf, _, _ = byname[name]
        yield name, cloud, cam, cfg, tn, tf, RENDERS
    # constant colour: every hit pixel renders exactly that colour (test_acceptance.py:349-362)
    _, cloud, cam, cfg, tn, tf, _, _ = byname["small_parallel_planes"]
    const = PointCloud(cloud.positions, np.tile([0.25, 0.5, 0.75], (cloud.count, 1)))
    yield "const_planes", const, cam, cfg, tn, tf, RENDERS[:3]
