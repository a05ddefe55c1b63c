# e2e (host buffers in / out) at several ray-chunk cuts: HP_E2E_CUTS=none is the one-pass path
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-parity"
for c in ${CUTS:-none 0.15,0.75}; do
  echo "== cuts $c"
  HP_E2E_CUTS=$c $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print(d['ms_per_step'], 'e2e %.3fM rays/s' % (e['value']/1e6), 'pinned %.3fM' % (e.get('pinned_inputs',{}).get('value',0)/1e6), 'view %.3fM' % (e.get('view',{}).get('value',0)/1e6))"
done
