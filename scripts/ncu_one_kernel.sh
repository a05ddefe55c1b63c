# ncu --set full of one kernel of one cfg2 frame: KREGEX=... (after a plain run)
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity"
$CMD > gpurun_out/plain_one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-1} -c 1 \
    -o gpurun_out/${OUT:-prof_one} $CMD > gpurun_out/ncu_one.log 2>&1
echo "ncu rc=$?"
