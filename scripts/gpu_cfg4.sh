# cfg4 radius sweep, parity-gated (device time; no e2e / cpu legs)
for wl in ${WLS:-cfg4 cfg4_d01}; do
  timeout 1500 python bench.py --workload $wl --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/g_$wl.log 2>&1; echo "$wl rc=$?"
  tail -c 1500 gpurun_out/g_$wl.log; echo
done
