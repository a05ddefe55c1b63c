# full ncu of one kernel (regex $1), -c ${2:-1}; plain run first
set -x
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity"
$CMD > gpurun_out/plain_one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$1" -c ${2:-1} \
    -o gpurun_out/prof_one $CMD > gpurun_out/ncu_one.log 2>&1
echo "ncu rc=$?"
tail -n 3 gpurun_out/ncu_one.log
