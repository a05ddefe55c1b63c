"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file, hdr, cur_line = None, None, None
agg = collections.defaultdict(lambda: [0, 0, collections.Counter(), ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) // 2:
        continue
    if r[0]:
        cur_line = (cur_file, r[0], r[1])
    if not r[2]:
        continue
    try:
        s = int(r[4] or 0)
        n = int(r[7] or 0)
    except ValueError:
        continue
    a = agg[cur_line[:2]]
    a[0] += s
    a[1] += n
    a[3] = cur_line[2]
    for k, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name and k < len(r):
            try:
                a[2][name[6:]] += int(r[k] or 0)
            except ValueError:
                pass
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"samples={tot} instructions={toti}")
for (f, l), (s, n, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    reasons = ",".join(f"{k}:{100*v//max(s,1)}" for k, v in st.most_common(3))
    print(f"{100*s/tot:5.1f}% {100*n/toti:5.1f}%i {f}:{l} [{reasons}] {src.strip()[:80]}")
