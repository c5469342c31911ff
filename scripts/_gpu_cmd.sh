timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
for c in c3 c5_t02 c5_t06 c5_t10 c5_t14 c5_t18 c5_t22 c5_t11 c5_t23; do timeout 200 python scripts/run_case.py $c --iters 5 --check; done > gpurun_out/cases.log 2>&1
