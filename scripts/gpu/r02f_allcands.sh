# every candidate of every BASELINE workload, timed (data for the planner's cost ranking)
for r in c1 c2a c2b c3 c4 c4s $(seq -f "c5_t%02g" 0 23); do
  timeout 600 python scripts/run_case.py $r --iters 6 > gpurun_out/cands_$r.log 2>&1; echo "$r rc=$? $(grep -c 'GB/s' gpurun_out/cands_$r.log)"
done
