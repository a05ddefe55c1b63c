"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run): build, full-CSR query + sample, the head path
with short heads (second-chance re-sort and full-path re-runs), the
operator shim, the renderer.  Checks the results against each other so a
sanitizer-perturbed run still has to be right."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_14044_b200 as hp  # noqa: E402
from paper_2404_14044_b200 import device as dv, pipeline  # noqa: E402

size = int(os.environ.get("SAN_SIZE", "48"))
dev = torch.device("cuda")
cloud = hp.generate_scene(hp.SceneSpec("parallel_planes", n=20_000, seed=3, plane_count=3, plane_gap=0.05,
                                       extent=0.8, noise=0.01))
cam = hp.scene_camera(size, size * 5 // 6, fov_deg=14)
cfg = hp.SearchConfig(hp.kernel_radius_for_min_radius(cam, 1.0, 0.04), hp.pixel_disc_radius(cam))
dirs, pixels = hp.ray_grid(cam)
m = len(dirs)
slopes = hp.radius_slopes(cam, pixels, cfg.kernel_radius)
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
rays = (up(pixels), up(dirs), up(np.full(m, 1.0)), up(np.full(m, 10.0)), up(slopes))
idx = dv.build(up(cloud.positions), cam, cfg.pad)
col = up(cloud.colors)
sc = hp.SamplerConfig()
full = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=False)
for want, whole in ((16, 16), (400, 512)):
    dv.PREFIX_WANT, dv.HEAD_WHOLE = want, whole
    head = pipeline._query_sample(idx, col, *rays, sc, True, None, prefix=True)
    for a, b in zip(head.samples, full.samples):
        assert torch.equal(a, b), "head path differs from the full path"
    print(f"want {want}: Q={head.Q} R={head.R} resorted={head.resorted} full-path={head.flagged}")
from paper_2404_14044_b200 import _kernels as K  # noqa: E402
rng = np.random.default_rng(0)
bk = rng.integers(0, 97, 5000).astype(np.int64)
cur = np.concatenate([[0], np.cumsum(np.bincount(bk, minlength=97))])[:-1].astype(np.int64)
out = np.zeros(5000, np.int64)
K.scatter_by_bucket(bk, np.arange(5000, dtype=np.int64), cur, out)
assert np.all(np.diff(out[np.argsort(bk, kind="stable")]) != 0)
torch.cuda.synchronize()
print("sanitize case ok", m, "rays")
