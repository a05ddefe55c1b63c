# ncu --set full of the head-path kernels of one cfg2 frame (after a plain run)
set -x
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity"
$CMD > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^(k_head_scan|k_head_sort|k_head_select|k_sample_plan|k_sample_exact)" -c 12 \
    -o gpurun_out/prof_head $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -n 5 gpurun_out/ncu_full.log
