"""Print one bench line's time, head re-sort / full-path counts, stages and kernels (stdin: bench output)."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
c = d["config"]
print(sys.argv[1] if len(sys.argv) > 1 else "", d["ms_per_step"], c.get("head_resorted_rays"), c.get("full_path_rays"))
print(" ", d.get("kernels_ms"))
