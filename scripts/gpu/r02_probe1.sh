# c4s candidates and an ncu capture of its tile_kernel, exported on the box
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tma_probe scripts/tma_probe.cu && /tmp/tma_probe > gpurun_out/tma_probe.log 2>&1
python scripts/run_case.py c4s --check > gpurun_out/c4s_cands.log 2>&1
P="kern=smem;kx=2;ky=1;tx=32;ty=64;order=0;occ=0;st=2;bp=1;vec=1"
python scripts/run_case.py c4s --plan "$P" --iters 3 > gpurun_out/c4s_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:tile_kernel -s 2 -c 1 -o /tmp/c4s_tile python scripts/run_case.py c4s --plan "$P" --iters 3 > gpurun_out/c4s_ncu.log 2>&1
ncu -i /tmp/c4s_tile.ncu-rep --page raw --csv > gpurun_out/c4s_tile_raw.csv
ncu -i /tmp/c4s_tile.ncu-rep --page details --csv > gpurun_out/c4s_tile_details.csv
cat gpurun_out/tma_probe.log
cat gpurun_out/c4s_cands.log
