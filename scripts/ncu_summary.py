"""Summarise an `ncu --set full` report into profiles/<name>.json: per launch
duration, DRAM bytes, grid, registers and active warps, plus the DRAM traffic
per library timing span (the names bench.py reports) for roofline.traffic.

usage: python scripts/ncu_summary.py gpurun_out/prof_full.ncu-rep profiles/r01_ncu_full.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
           "launch__block_size", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]

# library timing span (bench.py "kernels_ms" key) -> kernel launches it covers
SPANS = {
    "k_query_scan": ["k_query_scan"],
    "k_query_sort": ["k_query_sort<1024, 256>", "k_query_sort<2048, 512>"],
    "k_query_sort_large": ["k_query_sort<4096, 512>", "k_query_sort<8192, 1024>", "k_query_split",
                           "k_query_sort_parts<8192, 1024>"],
    "k_query_prefix": ["k_query_prefix<512, 128>", "k_query_prefix<1024, 256>"],
    "k_prefix_select": ["k_prefix_select<1024, 1024>"],
    "k_head_scan": ["k_head_scan"],
    "k_head_select": ["k_head_select<1024>"],
    "k_head_sort": ["k_head_sort<512, 128>", "k_head_sort<1024, 256>"],
    "k_query_bound": ["k_query_bound"],
    "k_mlp_agg": ["k_agg<8>"],
    "k_mlp_head": ["k_mlp_head"],
    "k_sample_plan": ["k_sample_plan"],
    "k_sample_exact": ["k_sample_exact"],
    "k_sample_retain": ["k_sample_retain"],
}


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    name = name.split("(")[0]
    return name.replace("void ", "").replace("hp::", "").strip()


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m in METRICS:
            if m not in hdr:
                continue
            v = r[hdr.index(m)].replace(",", "")
            u = units[hdr.index(m)]
            x = float(v) if v else 0.0
            if u == "Gbyte":
                x *= 1e9
            elif u == "Mbyte":
                x *= 1e6
            elif u == "Kbyte":
                x *= 1e3
            if u in ("ms",):
                x *= 1e3  # -> us
            elif u in ("ns",):
                x *= 1e-3
            d[m] = x
        launches.append(d)
    spans = {}
    for span, names in SPANS.items():
        sel = [d for d in launches
               if any(d["kernel"] == n or (d["kernel"].startswith(n) and ("<" in n or d["kernel"][len(n)] == "<"))
                      for n in names)]
        if not sel:
            continue
        # one span occurrence per frame: the longest capture of each kernel
        # (the first frame's query also launches a scan that only reports the
        # scratch it needs)
        best = {}
        for d in sel:
            if d["kernel"] not in best or d["gpu__time_duration.sum"] > best[d["kernel"]]["gpu__time_duration.sum"]:
                best[d["kernel"]] = d
        first = list(best.values())
        spans[span] = {"launches": [d["kernel"] for d in first],
                       "dram_bytes": sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in first),
                       "duration_us": sum(d["gpu__time_duration.sum"] for d in first)}
    json.dump({"report": rep, "metrics": METRICS, "launches": launches, "spans": spans}, open(out, "w"), indent=1)
    for k, v in spans.items():
        print(f"{k:20s} {v['duration_us']:9.1f} us  {v['dram_bytes'] / 1e9:7.3f} GB  {v['launches']}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
