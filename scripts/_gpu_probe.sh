timeout 600 python scripts/dbg_plans.py vec=3 > gpurun_out/dbg_plans.log 2>&1
for c in c5_t10 c5_t12 c2b c5_t00 c5_t04 c5_t19; do timeout 300 python scripts/run_case.py $c --iters 5 --check > gpurun_out/cands_$c.log 2>&1; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
