# final state of round 2: GPU suite, smoke, then the evidence set
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
bash scripts/gpu/r02d_final.sh
timeout 1200 python scripts/heuristic_gap.py > gpurun_out/heuristic_gap_after.log 2>&1; tail -1 gpurun_out/heuristic_gap_after.log
