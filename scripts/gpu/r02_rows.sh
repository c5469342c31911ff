timeout 1200 python -m pytest tests/test_gpu_rows.py -q -p no:cacheprovider -x > gpurun_out/rows_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/rows_tests.log
for c in c5_t04 c5_t01 c5_t05 c5_t19 p_suite_d3_132; do
  timeout 300 python scripts/run_case.py $c --iters 8 > gpurun_out/rows_$c.log 2>&1
  head -1 gpurun_out/rows_$c.log | cut -c1-70; grep -v "^#" gpurun_out/rows_$c.log | sort -k3 -n -r | head -2; echo "  bulk:"; grep "bulk=" gpurun_out/rows_$c.log | sort -k3 -n -r | head -3
done
