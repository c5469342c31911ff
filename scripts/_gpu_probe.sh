timeout 600 python scripts/dbg_plans.py vec= > gpurun_out/dbg_plans.log 2>&1
for c in c5_t15 c5_t06 c5_t12 c5_t08 c5_t14 c5_t02; do timeout 300 python scripts/run_case.py $c --iters 5 --check > gpurun_out/cands_$c.log 2>&1; done
