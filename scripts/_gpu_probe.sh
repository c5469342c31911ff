timeout 600 python scripts/dbg_plans.py vec= > gpurun_out/dbg_plans.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
