# one compute-sanitizer tool per call (TOOL=memcheck|racecheck|synccheck)
TOOL=${TOOL:-memcheck}
timeout 600 python scripts/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 --log-file gpurun_out/r02_sanitizer_$TOOL.log python scripts/sanitize_cases.py > gpurun_out/r02_sanitizer_${TOOL}_stdout.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/sanitize_plain.log; tail -12 gpurun_out/r02_sanitizer_$TOOL.log; tail -3 gpurun_out/r02_sanitizer_${TOOL}_stdout.log
