for c in c5_t20 c5_t02 c5_t18; do timeout 200 python scripts/run_case.py $c --iters 5 --check --top 14; done > gpurun_out/cases.log 2>&1
