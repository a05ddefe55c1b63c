"""Device time of hp_render (volume and knp) over the cfg2 frame's retained
samples (diagnostics for DESIGN.md; the image itself is not the bench metric)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_14044_b200 import device, pipeline  # noqa: E402
from paper_2404_14044_b200.sampler import SamplerConfig  # noqa: E402

w = bench.make_workload("cfg2")
dev = torch.device("cuda")
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
col = up(w["cloud"].colors)
fr = pipeline.frame_device(up(w["cloud"].positions), col, w["cam"], w["cfg"], up(w["pixels"]), up(w["dirs"]),
                           up(w["t_near"]), up(w["t_far"]), up(w["slopes"]), SamplerConfig(), False)
r_off, r_id, r_t, r_dist, _, r_alpha, _, r_color, _ = fr.samples
cam = w["cam"]
lib = device._lib.load(require_device=True)
pix, tf = up(w["pixels"]), up(w["t_far"])
owner = torch.empty(cam.width * cam.height, dtype=torch.int32, device=dev)
image = torch.zeros((cam.height, cam.width, 3), dtype=torch.float64, device=dev)
depth = torch.zeros((cam.height, cam.width), dtype=torch.float64, device=dev)
bg = (ctypes.c_double * 3)(0.0, 0.0, 0.0)
p = device._ptr
for mode, name in ((0, "volume"), (1, "knp")):
    ts = []
    for it in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        device._lib.check(lib.hp_render(mode, p(r_off), w["m"], p(r_id), p(r_t), p(r_dist), p(r_alpha), p(r_color),
                                        p(col), p(pix), 2, p(tf), 8, bg, cam.width, cam.height, p(owner), p(image),
                                        p(depth), device._stream()))
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    R = int(r_id.numel())
    print(f"hp_render {name}: {np.mean(ts):.3f} ms for m={w['m']} rays, R={R} samples")
