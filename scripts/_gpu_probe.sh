timeout 600 python scripts/dbg_plans.py vec=3 > gpurun_out/dbg_plans.log 2>&1
timeout 900 python bench.py --no-e2e --no-cpu > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
