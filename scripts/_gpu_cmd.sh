timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
L=paper_1603_02297_b200/_lib
for cp in "c5_t00 kern=smem;kx=2;ky=2;tx=64;ty=64;order=1;occ=0" "c5_t16 kern=smem;kx=2;ky=1;tx=64;ty=64;order=0;occ=0" "c5_t22 kern=smem;kx=1;ky=1;tx=16;ty=128;order=0;occ=0"; do
  set -- $cp
  timeout 300 python scripts/ab_libs.py $1 "$2" $L/libttb.so $L/libttb_mb1.so
done > gpurun_out/ab.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
