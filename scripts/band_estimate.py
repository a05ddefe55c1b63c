"""Estimate N-GPU row-band scaling on one GPU: time every rank's band alone
(the N-GPU step time is the max over ranks, plus the sample gather)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2404_14044_b200 import pipeline
from paper_2404_14044_b200.sampler import SamplerConfig
w = bench.make_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
dev = torch.device("cuda")
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
xyz, col = up(w["cloud"].positions), up(w["cloud"].colors)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
def timed(r0, r1, reps=5):
    rays = [up(w[k][r0:r1]) for k in ("pixels", "dirs", "t_near", "t_far", "slopes")]
    v = w["pixels"][r0:r1, 1]
    rows = (int(v.min()), int(v.max()) + 1) if r1 - r0 < w["m"] else None  # a band: only its rows' points
    ts = []
    for i in range(reps + 2):
        flush.fill_(1.0); torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); pipeline.frame_device(xyz, col, w["cam"], w["cfg"], *rays, SamplerConfig(), True, rows=rows); b.record()
        torch.cuda.synchronize()
        if i >= 2: ts.append(a.elapsed_time(b))
    return float(np.mean(ts))
t1 = timed(0, w["m"])
print("N=1 %.3f ms" % t1)
for n in (2, 4, 8):
    times = [timed(*bench.row_bands(w, n, k)) for k in range(n)]
    tm = max(times)
    print("N=%d band ms min %.3f max %.3f -> est %.1f M rays/s, efficiency %.2f" % (n, min(times), tm, w["m"] / tm / 1e3, t1 / (n * tm)))
if len(sys.argv) > 2:  # per-band detail at N = argv[2]
    from paper_2404_14044_b200.shard import row_costs
    n = int(sys.argv[2])
    rc = row_costs(w["cloud"].positions, w["cam"], w["cfg"].pad)
    for k in range(n):
        r0, r1 = bench.row_bands(w, n, k)
        W = w["cam"].width
        print("band", k, "rows", r0 // W, r1 // W, "cost %.3e" % rc[r0 // W:r1 // W].sum(), "ms %.3f" % timed(r0, r1))
