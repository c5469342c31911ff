# TMA L2 promotion sizes on c4s (32-byte runs of A at a 64-byte pitch) and a few rows; canary test
timeout 900 python -m pytest tests/test_gpu_canary.py -q -p no:cacheprovider > gpurun_out/canary.log 2>&1; echo "canary rc=$?"; tail -3 gpurun_out/canary.log
for l2 in 0 64 128 256; do
  echo "== TTB_TMA_L2=$l2"
  for c in c4s c3 c5_t15 c5_t18 c1; do
    TTB_TMA_L2=$l2 timeout 300 python scripts/run_case.py $c --iters 8 --filter kern=tma 2>&1 | grep -v "^#" | sort -k3 -n -r | head -1 | sed "s/^/$c /"
  done
done
