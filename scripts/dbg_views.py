"""Diagnostics: sampler path counters on one cfg3 view (needs a DEBUG=1 build,
e.g. HP_LIB pointing at it)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E401
import bench
import paper_2404_14044_b200 as hp
from paper_2404_14044_b200 import _lib, pipeline

cloud, views = bench.make_views(1)
v = views[0]
dev = torch.device("cuda")
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
xyz, col = up(cloud.positions), up(cloud.colors)
m = v["m"]
rays = [up(v["pixels"]), up(v["dirs"]), up(np.full(m, bench.T_NEAR)), up(np.full(m, bench.T_FAR)), up(v["slopes"])]
L = _lib.load()
for exact in (True, False):
    buf = (ctypes.c_int64 * 8)()
    for it in range(2):
        L.hp_sample_debug_counters(buf, 1)
        fr = pipeline.frame_device(xyz, col, v["cam"], v["cfg"], *rays, hp.SamplerConfig(), exact)
        torch.cuda.synchronize()
        L.hp_sample_debug_counters(buf, 0)
    print("exact_t_end", exact, "Q", fr.Q, "R", fr.R, "prefix", fr.prefix)
    print("  counters rays=%d fast=%d proved0=%d exact_evals=%d cand=%d bound=%d" % tuple(list(buf)[:6]))

# how many rays end with exactly zero transmittance (vs the proved ones above)
fr = pipeline.frame_device(xyz, col, v["cam"], v["cfg"], *rays, hp.SamplerConfig(), True)
t_end = fr.samples[8].cpu().numpy()
q = None
print("t_end == 0:", int((t_end == 0).sum()), "t_end > 0:", int((t_end > 0).sum()),
      "t_end > 1e-300:", int((t_end > 1e-300).sum()), "t_end == 1:", int((t_end == 1).sum()))
