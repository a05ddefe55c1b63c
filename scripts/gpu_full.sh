# tests + smoke + full bench line (e2e and cpu baseline included)
set -x
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; tail -c 3000 gpurun_out/bench_full.log; tail -c 1500 gpurun_out/bench_ref.log
