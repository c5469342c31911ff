# after the ranking pass: GPU suite, the heuristic choice against the tuned plan live
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 1200 python scripts/heuristic_gap.py > gpurun_out/heuristic_gap_after.log 2>&1; tail -32 gpurun_out/heuristic_gap_after.log | cut -c1-110
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
