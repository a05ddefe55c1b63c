# one compute-sanitizer tool per call: TOOL=memcheck|racecheck|synccheck
set -x
python scripts/sanitize_case.py > gpurun_out/san_plain.log 2>&1 && \
timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool ${TOOL} --error-exitcode 9 --print-limit 50 \
    python scripts/sanitize_case.py > gpurun_out/sanitize_${TOOL}.log 2>&1
echo "sanitizer rc=$?"
tail -n 8 gpurun_out/sanitize_${TOOL}.log
