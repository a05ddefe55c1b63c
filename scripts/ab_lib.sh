# cfg2 device time: the default library vs abl/var_*.so build variants (bench, no parity / e2e / cpu legs)
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
pr() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], {k:v for k,v in list(d['kernels_ms'].items())[:7]})"; }
for rep in 1 2; do
  echo "== base"; $B 2>/dev/null | pr
  for f in abl/var_*.so; do [ -f "$f" ] && { echo "== $f"; HP_LIB=$PWD/$f $B 2>/dev/null | pr; }; done
done
true
