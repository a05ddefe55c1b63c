import numpy as np, torch, bench, sys
from paper_2404_14044_b200 import device as dv
w = bench.make_workload("cfg2")
dev = torch.device("cuda")
up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
idx = dv.build(up(w["cloud"].positions), w["cam"], w["cfg"].pad)
q = dv.query(idx, *[up(w[k]) for k in ("pixels", "dirs", "t_near", "t_far", "slopes")])
off = q[0].cpu().numpy(); t = q[2].cpu().numpy()
qq = np.diff(off); hit = np.nonzero(qq > 64)[0]
rng = np.random.default_rng(0); sel = np.sort(rng.choice(hit, 3000, replace=False))
segs = [t[off[r]:off[r+1]] for r in sel]
np.savez_compressed("gpurun_out/tsegs.npz", lens=np.array([len(s) for s in segs]), t=np.concatenate(segs))
print("ok", len(segs))
