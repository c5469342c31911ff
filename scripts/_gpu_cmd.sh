B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-configs"
$B > gpurun_out/prof_plain.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "ttb_timed/" --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
P1="kern=smem;kx=2;ky=2;tx=64;ty=64;order=1;occ=0"
P2="kern=rt;mx=2;my=2;lx=4;kx=2;ky=2;order=0;occ=0"
timeout 120 python scripts/run_case.py c5_t00 --plan "$P1" --iters 3 > gpurun_out/p1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_kernel -s 2 -c 1 -o gpurun_out/prof_dense_t00 python scripts/run_case.py c5_t00 --plan "$P1" --iters 3 > gpurun_out/ncu1.log 2>&1
timeout 120 python scripts/run_case.py c3 --plan "$P2" --iters 3 > gpurun_out/p2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:rt_kernel -s 2 -c 1 -o gpurun_out/prof_rt_c3 python scripts/run_case.py c3 --plan "$P2" --iters 3 > gpurun_out/ncu2.log 2>&1
