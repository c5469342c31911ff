# GPU suite, then the final evidence set of round 2
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
bash scripts/gpu/r02d_final.sh
