# parity-gated bench lines of the named shapes (no e2e / cpu legs)
set -x
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g_cfg2.log 2>&1; echo "cfg2 rc=$?"
timeout 1200 python bench.py --workload cfg3 --views ${VIEWS:-16} --steps 2 --warmup 1 > gpurun_out/g_cfg3.log 2>&1; echo "cfg3 rc=$?"
timeout 1200 python bench.py --workload cfg4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g_cfg4.log 2>&1; echo "cfg4 rc=$?"
for f in g_cfg2 g_cfg3 g_cfg4; do echo "== $f"; tail -c 1200 gpurun_out/$f.log; echo; done
