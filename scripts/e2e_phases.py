"""Host-side phase times of pipeline.search_and_sample on cfg2 (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2404_14044_b200 import device, pipeline
from paper_2404_14044_b200.geometry import radius_slopes
from paper_2404_14044_b200.sampler import SamplerConfig
w = bench.make_workload("cfg2")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
P = dict(pos=pin(w["cloud"].positions), col=pin(w["cloud"].colors), pix=pin(w["pixels"]), dirs=pin(w["dirs"]),
         tn=pin(w["t_near"]), tf=pin(w["t_far"]))
dev = torch.device("cuda")
for it in range(4):
    T = [("start", time.perf_counter())]
    mark = lambda n: (torch.cuda.synchronize(), T.append((n, time.perf_counter())))
    xyz = P["pos"].to(dev, non_blocking=True); col = P["col"].to(dev, non_blocking=True); mark("h2d cloud")
    idx = device.build(xyz, w["cam"], w["cfg"].pad); mark("build")
    sl = radius_slopes(w["cam"], P["pix"].numpy(), w["cfg"].kernel_radius, w["cfg"].use_approx_radius); mark("host slopes")
    pix = P["pix"].to(dev, non_blocking=True); dirs = P["dirs"].to(dev, non_blocking=True)
    tn = P["tn"].to(dev, non_blocking=True); tf = P["tf"].to(dev, non_blocking=True)
    sld = torch.from_numpy(sl).to(dev); mark("h2d rays")
    q = device.query(idx, pix, dirs, tn, tf, sld); mark("query")
    s = device.sample(q[0], q[1], q[2], q[3], sld, SamplerConfig(), col, True); mark("sample")
    outs = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in s]; mark("alloc pinned")
    for o, x in zip(outs, s): o.copy_(x, non_blocking=True)
    mark("d2h")
    res = [o.numpy() for o in outs]; mark("numpy")
    print(" ".join(f"{b[0]}={1e3*(b[1]-a[1]):.2f}" for a, b in zip(T[:-1], T[1:])), f"total={1e3*(T[-1][1]-T[0][1]):.2f}")
t0 = time.perf_counter(); pipeline.search_and_sample(type("C", (), dict(positions=P["pos"], colors=P["col"]))(), w["cam"], w["cfg"], P["pix"], P["dirs"], P["tn"], P["tf"]); torch.cuda.synchronize(); print("search_and_sample", 1e3*(time.perf_counter()-t0))
