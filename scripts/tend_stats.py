import numpy as np, torch, bench, sys
from paper_2404_14044_b200 import pipeline
from paper_2404_14044_b200.sampler import SamplerConfig
w = bench.make_workload("cfg2")
dev = torch.device("cuda")
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
fr = pipeline.frame_device(up(w["cloud"].positions), up(w["cloud"].colors), w["cam"], w["cfg"], *[up(w[k]) for k in ("pixels","dirs","t_near","t_far","slopes")], SamplerConfig(), True)
te = fr.samples[8].cpu().numpy(); q = np.diff(fr.query[0].cpu().numpy())
hit = q > 0
print("hit", hit.sum(), "t_end==0", (te[hit] == 0).sum(), "t_end>0", (te[hit] > 0).sum())
nz = hit & (te > 0)
print("q of t_end>0 rays: mean", q[nz].mean(), "median", np.median(q[nz]), "sum", q[nz].sum(), "min t_end", te[nz].min(), "max", te[nz].max())
print("quantiles of t_end>0:", np.quantile(te[nz], [0.01, 0.1, 0.5, 0.9]))
