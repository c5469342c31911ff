timeout 600 python scripts/dbg_plans.py vec= > gpurun_out/dbg_plans.log 2>&1
python scripts/var_probe.py c5_t00 "kern=smem;kx=2;ky=2;tx=128;ty=128;order=0;occ=0;st=2;bp=1;vec=3" c5_t23 "kern=smem;kx=3;ky=1;tx=64;ty=36;order=0;occ=0;st=2;bp=1;vec=3" > gpurun_out/var.log 2>&1
python scripts/var_probe.py c5_t14 "kern=smem;kx=1;ky=1;tx=64;ty=64;order=0;occ=0;st=2;bp=1;vec=3" c5_t13 "kern=smem;kx=1;ky=1;tx=16;ty=128;order=0;occ=0;st=3;bp=1;vec=1" >> gpurun_out/var.log 2>&1
for c in c1 c5_t08 c5_t10 c5_t16; do timeout 300 python scripts/run_case.py $c --iters 5 --check --top 12 > gpurun_out/cands_$c.log 2>&1; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
