# GPU suite, then mixed kind pairs against the same rows in one kind
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -8 gpurun_out/gpu_tests.log
for spec in "c5_t00 ss" "c5_t00 sd" "c5_t16 ss" "c5_t16 sd" "c5_t09 dd" "c5_t09 ds" "c5_t21 dd" "c5_t21 ds" "c4 cc" "c4 cz" "c4 zz" "c4 zc" "c5_t23 dd" "c5_t23 ds"; do
  set -- $spec
  timeout 300 python scripts/run_case.py $1 --kinds $2 --iters 5 > gpurun_out/mixed_$1_$2.log 2>&1
  head -1 gpurun_out/mixed_$1_$2.log; grep -v "^#" gpurun_out/mixed_$1_$2.log | sort -k3 -n -r | head -2
done
