"""One N=8 row band of cfg2 on one GPU: frame device time vs the sum of its
kernels (the gap is launch / host-sync overhead), and the per-kernel split."""
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
n, k = (int(x) for x in (sys.argv[1:3] if len(sys.argv) > 2 else (8, 3)))
r0, r1 = bench.row_bands(w, n, k)
rays = [up(w[x][r0:r1]) for x in ("pixels", "dirs", "t_near", "t_far", "slopes")]
vv = w["pixels"][r0:r1, 1]
rows = (int(vv.min()), int(vv.max()) + 1) if n > 1 else None
tot, kern, cnt, stages = [], {}, {}, {}
for it in range(8):
    torch.cuda.synchronize()
    if it >= 3:
        _lib.timing_enable(True); _lib.timing_collect()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    timer = pipeline.StageTimer() if it >= 3 else None
    pipeline.device.TIMER = timer
    e0.record()
    pipeline.frame_device(xyz, col, w["cam"], w["cfg"], *rays, SamplerConfig(), True, timer=timer, rows=rows)
    e1.record(); torch.cuda.synchronize()
    pipeline.device.TIMER = None
    if timer is not None:
        for key, v in timer.spans().items():
            stages[key] = stages.get(key, 0.0) + v / 5
    if it >= 3:
        tot.append(e0.elapsed_time(e1))
        for key, (v, c) in _lib.timing_collect().items():
            kern[key] = kern.get(key, 0.0) + v / 5; cnt[key] = cnt.get(key, 0) + c / 5
        _lib.timing_enable(False)
ks = sum(kern.values())
print(f"band {k}/{n} rays {r1 - r0}: frame {np.mean(tot):.3f} ms, kernels {ks:.3f} ms, gap {np.mean(tot) - ks:.3f} ms, launches {sum(cnt.values()):.0f}")
for key, v in sorted(kern.items(), key=lambda x: -x[1]):
    print(f"   {key:28s} {v:.4f} ms  x{cnt[key]:.0f}")
print("   stages:", {k: round(v, 4) for k, v in stages.items()})
