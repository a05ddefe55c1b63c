"""Host-side phase times of pipeline.search_and_sample on cfg2 (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2404_14044_b200 import device, pipeline
from paper_2404_14044_b200.sampler import SamplerConfig
w = bench.make_workload("cfg2")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
P = dict(pos=pin(w["cloud"].positions), col=pin(w["cloud"].colors), pix=pin(w["pixels"]), dirs=pin(w["dirs"]),
         tn=pin(w["t_near"]), tf=pin(w["t_far"]))
dev = torch.device("cuda")
for it in range(5):
    T = [("start", time.perf_counter())]
    mark = lambda n: (torch.cuda.synchronize(), T.append((n, time.perf_counter())))
    xyz = P["pos"].to(dev, non_blocking=True); col = P["col"].to(dev, non_blocking=True); mark("h2d cloud")
    idx = device.build(xyz, w["cam"], w["cfg"].pad); mark("build")
    pix = P["pix"].to(dev, non_blocking=True); dirs = P["dirs"].to(dev, non_blocking=True)
    tn = P["tn"].to(dev, non_blocking=True); tf = P["tf"].to(dev, non_blocking=True); mark("h2d rays")
    sl = pipeline.host_slopes(w["cam"], P["pix"].numpy(), w["cfg"].kernel_radius, w["cfg"].use_approx_radius); mark("host slopes")
    sld = torch.from_numpy(sl).to(dev); mark("h2d slopes")
    q = device.query(idx, pix, dirs, tn, tf, sld, facts=True); mark("query")
    s = device.sample(q[0], q[1], q[2], q[3], sld, SamplerConfig(), col, True, facts=q[6]); mark("sample")
    outs = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in s]; mark("alloc pinned")
    for o, x in zip(outs, s): o.copy_(x, non_blocking=True)
    mark("d2h")
    print(" ".join(f"{b[0]}={1e3*(b[1]-a[1]):.2f}" for a, b in zip(T[:-1], T[1:])), f"total={1e3*(T[-1][1]-T[0][1]):.2f}")
C = type("C", (), dict(positions=P["pos"], colors=P["col"]))()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pipeline.search_and_sample(C, w["cam"], w["cfg"], P["pix"], P["dirs"], P["tn"], P["tf"]); torch.cuda.synchronize()
    print("search_and_sample", 1e3*(time.perf_counter()-t0))
