"""Generate tests/golden/render_*.npz by running the REFERENCE renderer.

Runs only in the dev container (the reference is not on the GPU box); the
reference is imported read-only from /root/reference/pkg/src with numba's
cache and Python bytecode redirected away from the source tree.

For a few golden cases (tests/golden_cases.py, the same seeded inputs) it
records the colour and depth images of ``render_volume`` and ``render_knp``
(renderer.py:138-192) over ``generate_rays(camera, t_near, t_far)``
(geometry.py:309-317) -- the reference's own full-view driver -- for several
render / sampler configurations, plus a constant-colour scene (the
acceptance suite's C8 identity, test_acceptance.py:349-362).

Usage:  python oracle/make_render_golden.py
"""

from __future__ import annotations

import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "hp_numba_cache"))
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from hashpoint import geometry as rgeo  # noqa: E402  (the reference)
from hashpoint import hash_index as ridx  # noqa: E402
from hashpoint import renderer as rren  # noqa: E402
from hashpoint import sampler as rsam  # noqa: E402
from hashpoint.cloud import PointCloud as RefCloud  # noqa: E402

import golden_cases  # noqa: E402
from golden_cases import render_cases  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def ref_camera(cam):
    return rgeo.Camera(np.array(cam.origin), np.array(cam.orientation), cam.focal_length,
                       cam.width, cam.height, cam.pixel_width, cam.pixel_height)


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, cloud, cam, cfg, tn, tf, configs in render_cases():
        rcam = ref_camera(cam)
        rcfg = rgeo.SearchConfig(cfg.kernel_radius, cfg.pixel_disc_radius, cfg.use_approx_radius)
        index = ridx.build(RefCloud(cloud.positions, cloud.colors), rcam, rcfg)
        rays = rgeo.generate_rays(rcam, tn, tf)
        rec = {"positions_sha": golden_cases_digest(cloud.positions)}
        for tag, mode, bg, knp_k, sampler in configs:
            rc = rren.RenderConfig(mode=mode, background=bg, knp_k=knp_k)
            sc = rsam.SamplerConfig(**golden_cases.SAMPLERS[sampler])
            img = rren.render(index, rays, rcfg, sc, rc)
            rec[f"{tag}_color"] = img.color
            rec[f"{tag}_depth"] = img.depth
            rec[f"{tag}_tnear_tfar"] = np.array([img.t_near, img.t_far])
        path = os.path.join(OUT, f"render_{name}.npz")
        np.savez_compressed(path, **rec)
        print("wrote", path, sorted(rec))


def golden_cases_digest(a):
    import hashlib
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


if __name__ == "__main__":
    main()
