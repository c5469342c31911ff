# whole-column candidates + prefetched tile claims: parity, then the rows they touch
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_canary.py tests/test_gpu_robustness.py -q -x -m gpu -p no:cacheprovider > gpurun_out/exp2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp2_tests.log
for r in c5_t14 c5_t06 c5_t22 c5_t00 c5_t07 c5_t13 c1; do
  timeout 600 python scripts/run_case.py $r --iters 8 --check > gpurun_out/exp2_$r.log 2>&1
  echo "== $r rc=$?"; grep "GB/s" gpurun_out/exp2_$r.log | sort -k3 -n -r | head -4; grep -c MISMATCH gpurun_out/exp2_$r.log
done
