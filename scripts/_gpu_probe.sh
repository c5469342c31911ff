timeout 900 python bench.py --no-e2e --no-cpu --no-configs > gpurun_out/bench_clk.log 2>&1; echo rc=$? >> gpurun_out/bench_clk.log
head -3 gpurun_out/clocks_rank0.csv > gpurun_out/clk_head.txt
