timeout 1200 python -m pytest tests/test_gpu_tma.py -q -p no:cacheprovider -k "bulk_tile" > gpurun_out/ts_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ts_tests.log
for c in c5_t14 c5_t06 c5_t09 c5_t18; do
  timeout 300 python scripts/run_case.py $c --iters 8 > gpurun_out/ts_$c.log 2>&1
  head -1 gpurun_out/ts_$c.log; grep -v "^#" gpurun_out/ts_$c.log | sort -k3 -n -r | head -2; echo "  best ts:"; grep "ts=" gpurun_out/ts_$c.log | sort -k3 -n -r | head -2
done
