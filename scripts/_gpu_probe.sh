timeout 600 python scripts/dbg_plans.py xp= > gpurun_out/dbg_plans.log 2>&1
for c in c5_t18 c5_t08; do timeout 300 python scripts/run_case.py $c --iters 5 --check > gpurun_out/cands_$c.log 2>&1; done
