"""Per-source-line instruction / stall-sample totals of one kernel from an
`ncu --page source --csv --print-source cuda,sass` dump (file path blocks)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, out, hdr = None, [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    ci = hdr.index("Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        out.append((cur, r[0], r[1], float(r[ci]), float(r[si])))
    except ValueError:
        pass
ti = sum(o[3] for o in out)
ts = sum(o[4] for o in out)
print(f"total warp instructions {ti:.4g}, stall samples {ts:.4g}")
for f, ln, src, i, s in sorted(out, key=lambda o: -o[3])[:n_top]:
    print(f"{f}:{ln:>5} inst {100 * i / ti:5.1f}%  samples {100 * s / ts:5.1f}%  {src.strip()[:90]}")
