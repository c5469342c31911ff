timeout 600 python scripts/dbg_plans.py vec= > gpurun_out/dbg_plans.log 2>&1
for c in c1 c5_t00 c5_t22 c5_t03 c5_t13 c5_t20 c4 c2a; do timeout 300 python scripts/run_case.py $c --iters 5 --check > gpurun_out/cands_$c.log 2>&1; done
