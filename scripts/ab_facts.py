"""A/B: frame time with and without the query->sampler facts (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2404_14044_b200 import _lib, device, pipeline
from paper_2404_14044_b200.sampler import SamplerConfig
w = bench.make_workload("cfg2")
dev = torch.device("cuda")
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
xyz, col = up(w["cloud"].positions), up(w["cloud"].colors)
rays = [up(w[k]) for k in ("pixels", "dirs", "t_near", "t_far", "slopes")]
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
def frame(facts):
    idx = device.build(xyz, w["cam"], w["cfg"].pad)
    q = device.query(idx, *rays, facts=facts)
    return device.sample(q[0], q[1], q[2], q[3], rays[4], SamplerConfig(), col, True, facts=q[6] if facts else None)
res = {True: [], False: []}
_lib.timing_enable(True)
for it in range(16):
    f = bool(it % 2)
    flush.fill_(1.0)
    torch.cuda.synchronize()
    _lib.timing_collect()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); frame(f); b.record(); torch.cuda.synchronize()
    k = _lib.timing_collect()
    if it >= 4:
        res[f].append((a.elapsed_time(b), k))
for f in (False, True):
    ms = [x[0] for x in res[f]]
    ks = {}
    for _, k in res[f]:
        for n, (v, c) in k.items(): ks[n] = ks.get(n, 0) + v / len(res[f])
    print("facts", f, "frame ms %.3f" % np.mean(ms), {n: round(v, 3) for n, v in sorted(ks.items(), key=lambda x: -x[1])})
