CMD="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity"
$CMD > gpurun_out/plain_cfg5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^k_agg|^k_mlp_head" -s 2 -c 2 \
    -o gpurun_out/${OUT:-prof_mlp} $CMD > gpurun_out/ncu_mlp.log 2>&1
echo "ncu rc=$?"
