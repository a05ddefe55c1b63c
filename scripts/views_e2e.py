"""Per-call wall time of pipeline.search_and_sample_views on cfg3 views
(host-side timeline diagnostics: pinned allocation, copies, per-view syncs)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2404_14044_b200 import pipeline  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cloud, views = bench.make_views(n)
cams, cfgs = [v["cam"] for v in views], [v["cfg"] for v in views]
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = pipeline.search_and_sample_views(cloud, cams, cfgs, bench.T_NEAR, bench.T_FAR)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"call {it}: {1e3 * (t1 - t0):.1f} ms, {sum(x.nbytes for o in out.values() for x in o) / 1e9:.2f} GB out",
          flush=True)
for k in range(3):
    t0 = time.perf_counter()
    x = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    print(f"pinned 1 GiB alloc: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del x
