set -x
for V in "-DHP_STAGE_FILL=256 -DHP_SCAN_MINB=5" "-DHP_STAGE_FILL=384 -DHP_SCAN_MINB=4" ""; do
  make -s -C paper_2404_14044_b200/csrc EXTRA="$V" -B > /dev/null 2>&1
  echo "== $V" >> gpurun_out/ab.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | grep -o '"ms_per_step": [0-9.]*\|"k_query_scan": [0-9.]*\|"parity_gate": "[a-z]*' >> gpurun_out/ab.log
done
cat gpurun_out/ab.log
