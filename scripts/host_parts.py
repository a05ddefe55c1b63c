"""Host-side cost of issuing the e2e uploads (diagnostics)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch, bench
w = bench.make_workload("cfg2")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
pix = pin(w["pixels"]); dirs = pin(w["dirs"])
print("pinned", pix.is_pinned(), dirs.is_pinned())
dev = torch.device("cuda")
side = torch.cuda.Stream()
for it in range(4):
    T = [time.perf_counter()]
    with torch.cuda.stream(side):
        a = pix.to(dev, dtype=torch.int64, non_blocking=True)
    T.append(time.perf_counter())
    with torch.cuda.stream(side):
        b = dirs.to(dev, non_blocking=True)
    T.append(time.perf_counter())
    c = torch.empty(dirs.shape, dtype=dirs.dtype, device=dev); T.append(time.perf_counter())
    c.copy_(dirs, non_blocking=True); T.append(time.perf_counter())
    d = dirs.to(dev, non_blocking=True); T.append(time.perf_counter())
    torch.cuda.synchronize()
    print(" ".join("%.3f" % (1e3*(b-a)) for a, b in zip(T[:-1], T[1:])))
