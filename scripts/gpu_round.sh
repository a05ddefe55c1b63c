# full evidence run: tests, smoke, the default bench line, the reference arm, the named shapes
set -x
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 1200 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "cfg2 rc=$?"
timeout 1200 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 1800 python bench.py --workload cfg3 --steps 2 --warmup 1 > gpurun_out/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"
timeout 1200 python bench.py --workload cfg4 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; echo "cfg4 rc=$?"
timeout 1500 python bench.py --workload cfg4_d01 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_d01.log 2>&1; echo "cfg4_d01 rc=$?"
timeout 1200 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1; echo "cfg5 rc=$?"
timeout 1500 python bench.py --workload cfg4_d02 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4_d02.log 2>&1; echo "cfg4_d02 rc=$?"
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
for f in bench_cfg2 bench_ref bench_cfg3 bench_cfg4 bench_cfg4_d01 bench_cfg5 bench_cfg4_d02; do echo "== $f"; tail -c 600 gpurun_out/$f.log; echo; done
