set -x
for c in c1 c2a c3 c4 c4s c5_t00 c5_t04 c5_t08 c5_t12 c5_t15 c5_t22; do timeout 120 python scripts/run_case.py $c --iters 5 --check; done > gpurun_out/cases.log 2>&1
P1="kern=smem;kx=1;ky=1;tx=79;ty=51;order=0;occ=0"
P2="kern=rt;mx=4;my=4;lx=8;kx=1;ky=1;order=1;occ=0"
timeout 120 python scripts/run_case.py c5_t00 --plan "$P1" --iters 3 > gpurun_out/p1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:smem_kernel -s 2 -c 1 -o gpurun_out/prof_smem_t00 python scripts/run_case.py c5_t00 --plan "$P1" --iters 3 > gpurun_out/ncu1.log 2>&1
timeout 120 python scripts/run_case.py c1 --plan "$P2" --iters 3 > gpurun_out/p2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:rt_kernel -s 2 -c 1 -o gpurun_out/prof_rt_c1 python scripts/run_case.py c1 --plan "$P2" --iters 3 > gpurun_out/ncu2.log 2>&1
