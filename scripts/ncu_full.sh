# full ncu sections for the hot kernels of one frame (run after a plain run exits 0)
set -x
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity"
$CMD > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^(k_query_scan|k_query_sort|k_query_prefix|k_prefix_select|k_sample_plan|k_sample_exact|k_sample_retain)$" -c 20 \
    -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -n 5 gpurun_out/ncu_full.log
