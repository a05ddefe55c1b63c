"""Diagnostics: sampler path counters and per-stage timing on a workload (counters need `make -C paper_2404_14044_b200/csrc DEBUG=1`)."""
import ctypes, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2404_14044_b200 import _lib, device as dv, pipeline
w = bench.make_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
dev = torch.device("cuda")
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
xyz, col = up(w["cloud"].positions), up(w["cloud"].colors)
rays = [up(w[k]) for k in ("pixels", "dirs", "t_near", "t_far", "slopes")]
import paper_2404_14044_b200 as hp
L = _lib.load()
for exact in (True, False):
    for it in range(2):
        buf = (ctypes.c_int64 * 8)()
        L.hp_sample_debug_counters(buf, 1)
        t = pipeline.StageTimer(); dv.TIMER = t
        fr = pipeline.frame_device(xyz, col, w["cam"], w["cfg"], *rays, hp.SamplerConfig(), exact, t)
        dv.TIMER = None
        sp = t.spans()
        L.hp_sample_debug_counters(buf, 0)
    print("exact_t_end", exact, {k: round(v, 3) for k, v in sp.items()})
    print("  counters rays=%d fast=%d proved0=%d exact_evals=%d cand=%d sum_jstar=%d" % tuple(list(buf)[:6]))
