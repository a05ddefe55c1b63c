import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch, bench
from paper_2404_14044_b200 import pipeline, device
w = bench.make_workload("cfg2")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
C = type("C", (), dict(positions=pin(w["cloud"].positions), colors=pin(w["cloud"].colors)))()
P = dict(pix=pin(w["pixels"]), dirs=pin(w["dirs"]), tn=pin(w["t_near"]), tf=pin(w["t_far"]))
# monkeypatch marks
evs = []
def mark(name):
    e = torch.cuda.Event(enable_timing=True); e.record(); evs.append((name, e, time.perf_counter()))
orig_query, orig_sample, orig_build = device.query_prefix, device.sample_prefix, device.build
def q(*a, **k):
    mark("query>"); r = orig_query(*a, **k); mark("query<"); return r
def s(*a, **k):
    mark("sample>"); r = orig_sample(*a, **k); mark("sample<"); return r
def b(*a, **k):
    mark("build>"); r = orig_build(*a, **k); mark("build<"); return r
device.query_prefix, device.sample_prefix, device.build = q, s, b
for it in range(6):
    evs.clear(); torch.cuda.synchronize(); mark("start")
    out = pipeline.search_and_sample(C, w["cam"], w["cfg"], P["pix"], P["dirs"], P["tn"], P["tf"])
    mark("end"); torch.cuda.synchronize()
    t0g, t0h = evs[0][1], evs[0][2]
    print(" ".join(f"{n}:gpu{t0g.elapsed_time(e):.2f}/host{1e3*(h-t0h):.2f}" for n, e, h in evs[1:]))
