# ncu evidence of the final build: the launch list of one cfg2 frame (cold, serialised; compare shares)
# and --set full of the top kernels (after a plain run of the same command)
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity"
$CMD > gpurun_out/plain_ncu.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/plain_ncu2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^(k_head_scan|k_head_sort|k_head_select|k_sample_plan|k_sample_exact|k_query_bound)" -c 14 \
    -o gpurun_out/prof_r02 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
C5="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity"
$C5 > gpurun_out/plain_ncu3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^(k_agg|k_mlp_head)" -s 2 -c 2 \
    -o gpurun_out/prof_r02_mlp $C5 > gpurun_out/ncu_mlp.log 2>&1
echo "mlp rc=$?"
