"""Timeline of pipeline.search_and_sample on cfg2 at several ray-chunk counts
(host timestamps + device events; diagnostics for the overlapped copies)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2404_14044_b200 import pipeline
w = bench.make_workload(os.environ.get("WL", "cfg2"))
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
if os.environ.get("INPUT", "numpy") == "pinned":
    C = type("C", (), dict(positions=pin(w["cloud"].positions), colors=pin(w["cloud"].colors)))()
    P = [pin(w[k]) for k in ("pixels", "dirs", "t_near", "t_far")]
else:
    C, P = w["cloud"], [w[k] for k in ("pixels", "dirs", "t_near", "t_far")]
T = []
orig_qs, orig_hb, orig_sl, orig_b = pipeline._query_sample, pipeline._host_buffers, pipeline.host_slopes, pipeline.device.build
def sl(*a, **k):
    T.append(("sl+", time.perf_counter())); r = orig_sl(*a, **k); T.append(("sl-", time.perf_counter())); return r
def bd(*a, **k):
    T.append(("build", time.perf_counter())); return orig_b(*a, **k)
pipeline.host_slopes, pipeline.device.build = sl, bd
orig_h2d, orig_up = pipeline._h2d, pipeline._h2d_async
def h2d(*a, **k):
    T.append(("h2d+", time.perf_counter())); r = orig_h2d(*a, **k); T.append(("h2d-", time.perf_counter())); return r
pipeline._h2d = h2d
def s2h(*a, **k):
    T.append(("s2h+", time.perf_counter())); r = orig_s2h(*a, **k); T.append(("s2h-", time.perf_counter())); return r
orig_s2h = pipeline._samples_to_host
pipeline._samples_to_host = s2h
def qs(*a, **k):
    T.append(("qs+", time.perf_counter())); r = orig_qs(*a, **k); T.append(("qs-", time.perf_counter())); return r
def hb(*a, **k):
    T.append(("hb+", time.perf_counter())); r = orig_hb(*a, **k); T.append(("hb-", time.perf_counter())); return r
pipeline._query_sample, pipeline._host_buffers = qs, hb
for chunks in os.environ.get("CUTS", "none 0.15,0.75").split():
    pipeline.E2E_CUTS = tuple(float(x) for x in chunks.split(",")) if chunks != "none" else ()
    for it in range(5):
        T.clear()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = pipeline.search_and_sample(C, w["cam"], w["cfg"], *P)
        t1 = time.perf_counter()
        if it >= 3:
            print(f"chunks={chunks} total {1e3 * (t1 - t0):.2f} ms :", " ".join(f"{n}@{1e3 * (t - t0):.2f}" for n, t in T))
