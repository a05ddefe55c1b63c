# ncu --set full of one k_sample_exact launch of a cfg3 batch (after a plain run)
CMD="python bench.py --workload cfg3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-parity"
$CMD > gpurun_out/plain_cfg3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sample_exact" -s 3 -c 1 \
    -o gpurun_out/${OUT:-prof_exact3} $CMD > gpurun_out/ncu_exact3.log 2>&1
echo "ncu rc=$?"
