timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
for c in c4s c5_t00 c5_t02 c5_t06 c5_t08 c5_t10 c5_t12 c5_t14 c5_t16 c5_t18 c5_t20 c5_t22; do timeout 120 python scripts/run_case.py $c --iters 5 --check; done > gpurun_out/cases.log 2>&1
