# cfg3 (16 views) and cfg2 under head settings PAIRS="want:whole ..."
for p in ${PAIRS:-400:512}; do
  echo "== $p"
  HP_PREFIX_WANT=${p%%:*} HP_HEAD_WHOLE=${p##*:} python bench.py --workload cfg3 --views 16 --steps 2 --warmup 1 --no-parity 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('cfg3', d['ms_per_step'], c['head_resorted_rays'], c['full_path_rays'], {k:v for k,v in list(d['kernels_ms'].items())[:6]})"
  HP_PREFIX_WANT=${p%%:*} HP_HEAD_WHOLE=${p##*:} python bench.py --steps 10 --warmup 3 --no-parity --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', d['ms_per_step'], {k:v for k,v in list(d['kernels_ms'].items())[:8]})"
done
