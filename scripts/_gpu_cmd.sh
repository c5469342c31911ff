P1="kern=smem;kx=2;ky=2;tx=64;ty=64;order=1;occ=0"
timeout 120 python scripts/run_case.py c5_t00 --plan "$P1" --iters 3 > gpurun_out/p1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:smem -s 2 -c 1 -o gpurun_out/prof_smem3_t00 python scripts/run_case.py c5_t00 --plan "$P1" --iters 3 > gpurun_out/ncu1.log 2>&1
