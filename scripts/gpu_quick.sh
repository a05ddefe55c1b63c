# smoke + the -m gpu suite + one short bench line (no e2e / cpu baseline)
set -x
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -n 3 gpurun_out/smoke.log; tail -n 30 gpurun_out/pytest_gpu.log; tail -c 2500 gpurun_out/bench.log
