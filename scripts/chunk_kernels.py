"""Per-kernel device time of cfg2 run as one pass vs ray chunks (diagnostics:
where the per-chunk overhead goes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2404_14044_b200 import _lib, pipeline
from paper_2404_14044_b200.sampler import SamplerConfig
w = bench.make_workload("cfg2")
dev = torch.device("cuda")
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
xyz, col = up(w["cloud"].positions), up(w["cloud"].colors)
rays = [up(w[k]) for k in ("pixels", "dirs", "t_near", "t_far", "slopes")]
m = w["m"]
def run(cuts, reps=4):
    tot, kern = [], {}
    for it in range(reps + 2):
        torch.cuda.synchronize()
        if it >= 2:
            _lib.timing_enable(True); _lib.timing_collect()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        idx = pipeline.device.build(xyz, w["cam"], w["cfg"].pad)
        per = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            ea = torch.cuda.Event(enable_timing=True); eb = torch.cuda.Event(enable_timing=True)
            ea.record()
            pipeline._query_sample(idx, col, *[r[a:b] for r in rays], SamplerConfig(), True, None)
            eb.record(); per.append((ea, eb))
        e1.record(); torch.cuda.synchronize()
        if it >= 2:
            tot.append([e0.elapsed_time(e1)] + [x.elapsed_time(y) for x, y in per])
            for k, (v, c) in _lib.timing_collect().items():
                kern[k] = kern.get(k, 0.0) + v / reps
            _lib.timing_enable(False)
    t = np.mean(np.array(tot), axis=0)
    print("cuts", [round(c / m, 3) for c in cuts], "total %.2f ms, chunks" % t[0], np.round(t[1:], 2))
    print("   ", {k: round(v, 3) for k, v in sorted(kern.items(), key=lambda x: -x[1])[:14]})
run([0, m])
run([0, int(0.7 * m), m])
run([0, int(0.15 * m), int(0.75 * m), m])
