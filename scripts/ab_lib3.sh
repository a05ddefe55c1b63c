# cfg2 + cfg3 (16 views) device time: the default library vs abl/var_*.so
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
pr() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], {k:v for k,v in list(d['kernels_ms'].items())[:7]})"; }
for f in base abl/var_*.so; do
  L=""; [ "$f" != base ] && L=$PWD/$f
  echo "== $f"; HP_LIB=$L $B 2>/dev/null | pr
  HP_LIB=$L python bench.py --workload cfg3 --views 16 --steps 2 --warmup 1 --no-parity --no-e2e --no-cpu-baseline 2>/dev/null | pr
done
true
