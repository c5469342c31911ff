# final evidence of round 2: reference arm, engine arm, 2 ranks sharing the GPU (gloo),
# launch list of the timed region, ncu --set full of the kernels new since the last set, suite
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; echo "ref rc=$?"
timeout 1200 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
timeout 1200 python bench.py --gpus 2 --steps 3 --no-configs --no-cpu --no-e2e > gpurun_out/r02_bench_2rank_gloo.json 2> gpurun_out/r02_bench_2rank_gloo.err; echo "2rank rc=$?"
timeout 900 python bench.py --steps 1 --no-configs --no-cpu --no-e2e > gpurun_out/r02_launch_plain.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "ttb_timed/" --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --no-configs --no-cpu --no-e2e > gpurun_out/r02_launch_ncu.log 2>&1; echo "ncu rc=$?"
cap() {  # name case plan kernel-regex
  python scripts/run_case.py $2 --plan "$3" --iters 2 > gpurun_out/ncu_$1_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none -k regex:$4 -s 1 -c 1 -o /tmp/ncu_$1 \
      python scripts/run_case.py $2 --plan "$3" --iters 2 > gpurun_out/ncu_$1.log 2>&1 && \
  ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv
  echo "$1 rc=$?"; rm -f /tmp/ncu_$1.ncu-rep
}
cap btile_t14w c5_t14 "kern=smem;kx=1;ky=1;tx=60;ty=197;order=0;occ=0;st=2;bp=1;vec=3;ts=1" btile_kernel
cap btile_t07b c5_t07 "kern=smem;kx=1;ky=1;tx=32;ty=64;order=0;occ=0;st=2;bp=1;vec=3;ts=2" btile_kernel
cap btile_t00 c5_t00 "kern=smem;kx=2;ky=2;tx=128;ty=128;order=1;occ=0;st=2;bp=1;vec=3" btile_kernel
cap rowcopy_t04 c5_t04 "kern=copy;v=1;kx=0;ky=0;tx=1;ty=1;order=0;occ=0;bulk=32;st=3" rowcopy_kernel
cap rowcopy_t19 c5_t19 "kern=copy;v=1;kx=0;ky=0;tx=1;ty=1;order=0;occ=0;bulk=16;st=4" rowcopy_kernel
timeout 1500 python scripts/suite.py --ref --verify --csv gpurun_out/r02_suite_200MiB_s.csv > gpurun_out/r02_suite_200MiB_s.log 2>&1
echo "suite rc=$?"; tail -4 gpurun_out/r02_suite_200MiB_s.log
