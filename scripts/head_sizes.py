"""k_head_sort / k_head_select device time on one cfg2 frame at several
(want, whole) head sizes (diagnostics for the head length trade-off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2404_14044_b200 import _lib, device as dv
w = bench.make_workload(os.environ.get("WL", "cfg2"))
dev = torch.device("cuda")
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
idx = dv.build_layout(up(w["cloud"].positions), w["cam"], w["cfg"].pad)
rays = [up(w[k]) for k in ("pixels", "dirs", "t_near", "t_far", "slopes")]
for want, whole in ((400, 512), (400, 1024), (1024, 1024), (512, 512), (700, 1024)):
    for it in range(3):
        _lib.timing_enable(True); _lib.timing_collect()
        pre = dv.query_prefix(idx, *rays, want=want, whole=whole)
        torch.cuda.synchronize()
        t = _lib.timing_collect(); _lib.timing_enable(False)
        hl = int(pre.length.sum())
        del pre
    print(want, whole, "head entries %.3g" % hl, {k: round(v[0], 3) for k, v in t.items() if "head" in k})
