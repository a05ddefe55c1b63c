"""Per-kernel share of one bench frame from an ncu launch list
(--metrics gpu__time_duration.sum --csv of bench.py --steps 1 --warmup 1).
Frames start at the build's first kernel (k_project); the timed frame is the
second one (the bench runs the warm-up frame, the timed frame, then one more
untimed frame for its byte counts)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
launch = []
for r in rows[1:]:
    name = r[ki].replace("<unnamed>::", "").replace("(anonymous namespace)::", "").replace("void ", "")
    name = name.replace("hp::", "").split("(")[0]
    launch.append((name, float(r[vi].replace(",", ""))))
starts = [i for i, (nm, _) in enumerate(launch) if nm.startswith("k_project")]
if len(starts) >= 2:
    frame = launch[starts[1]:starts[2] if len(starts) > 2 else len(launch)]
    where = "the timed frame (second of the launch list)"
else:
    frame = launch[len(launch) // 2:]
    where = "second half of the launch list"
s = sum(v for _, v in frame)
agg = collections.Counter()
for nm, v in frame:
    agg[nm] += v
out = [f"frame = {where}: {len(frame)} launches, {s / 1e6:.3f} ms serialised "
       f"(ncu, cold caches, --clock-control none)"]
for k, v in agg.most_common():
    out.append(f"{k[:60]:60s} {v / 1e3:9.1f} us {100 * v / s:6.1f}%")
print("\n".join(out))
