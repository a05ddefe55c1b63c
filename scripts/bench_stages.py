"""Print one bench line's time and stages (stdin: bench output)."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(sys.argv[1] if len(sys.argv) > 1 else "", d["ms_per_step"], d["config"].get("head_resorted_rays"))
print(" ", {k: v for k, v in d.get("stages_ms", {}).items()})
