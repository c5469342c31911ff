timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo rc=$? >> gpurun_out/bench_full.log
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "ttb_timed/" --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-configs > gpurun_out/ncu_launch.log 2>&1; echo rc=$? >> gpurun_out/ncu_launch.log
bash scripts/prof_rows.sh c5_t00 "kern=smem;kx=2;ky=2;tx=128;ty=128;order=0;occ=0;st=2;bp=1;vec=3" c5_t22 "kern=smem;kx=1;ky=1;tx=48;ty=64;order=0;occ=0;st=2;bp=1;vec=3"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
