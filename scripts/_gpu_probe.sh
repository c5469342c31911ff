timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for c in c5_t00 c5_t19 c5_t22; do timeout 300 python scripts/run_case.py $c --iters 5 --check --top 3 > gpurun_out/cands_$c.log 2>&1; done
