# A/B of head-path variants on cfg2 (bench device time); PAIRS="want:whole ..."; variant libraries in abl/
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
run() { echo "== $1"; shift; env "$@" $B 2>&1 | python -c "
import json,sys
lines=sys.stdin.read().strip().splitlines()
try:
    d=json.loads(lines[-1]); print(d['ms_per_step'], d['config']['prefix_flagged_rays'], {k:v for k,v in d['kernels_ms'].items() if v>0.2})
except Exception: print('\n'.join(lines[-6:]))"; }
run base HP_LIB=$PWD/paper_2404_14044_b200/libhp_b200.so
for p in ${PAIRS:-400:512}; do
  run "want:whole=$p" HP_PREFIX_WANT=${p%%:*} HP_HEAD_WHOLE=${p##*:}
done
for f in abl/var_*.so; do [ -f "$f" ] && run $(basename $f) HP_LIB=$PWD/$f; done
true
