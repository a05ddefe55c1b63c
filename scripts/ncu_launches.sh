# per-kernel launch list of one bench frame (cold-cache, serialised; compare shares)
set -x
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"
tail -n 3 gpurun_out/ncu.log
