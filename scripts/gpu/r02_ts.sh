timeout 1500 python -m pytest tests/test_gpu_tma.py tests/test_gpu_robustness.py tests/test_gpu_canary.py -q -p no:cacheprovider -x > gpurun_out/ts_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ts_tests.log
for c in c5_t14 c5_t07 c5_t23; do
  timeout 300 python scripts/run_case.py $c --iters 8 --filter "ts=" > gpurun_out/ts_$c.log 2>&1
  head -1 gpurun_out/ts_$c.log | cut -c1-60; grep -v "^#" gpurun_out/ts_$c.log | sort -k3 -n -r | head -2
done
