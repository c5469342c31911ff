# first TMA tile run: parity tests, then every candidate on the aligned workloads
timeout 900 python -m pytest tests/test_gpu_tma.py -x -q > gpurun_out/tma_tests.log 2>&1
echo "tests rc=$?"
tail -30 gpurun_out/tma_tests.log
for c in c1 c2a c3 c4 c4s c5_t15 c5_t18 c5_t23 c5_t02 c5_t20; do
  timeout 300 python scripts/run_case.py $c --check --iters 5 > gpurun_out/tma_case_$c.log 2>&1
  grep -E "^#|tma" gpurun_out/tma_case_$c.log | head -12
  sort -k3 -n -r gpurun_out/tma_case_$c.log | grep -v "^#" | head -3
done
