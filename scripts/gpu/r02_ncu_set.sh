# ncu --set full of each kernel family on its BASELINE row, exported on the box (raw + details CSV)
cap() {  # name case plan kernel-regex
  python scripts/run_case.py $2 --plan "$3" --iters 2 > gpurun_out/ncu_$1_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none -k regex:$4 -s 1 -c 1 -o /tmp/ncu_$1 \
      python scripts/run_case.py $2 --plan "$3" --iters 2 > gpurun_out/ncu_$1.log 2>&1 && \
  ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv && \
  ncu -i /tmp/ncu_$1.ncu-rep --page details --csv > gpurun_out/ncu_$1_details.csv
  echo "$1 rc=$?"; rm -f /tmp/ncu_$1.ncu-rep
}
cap tma_c3 c3 "kern=tma;kx=2;ky=1;tx=240;ty=16;order=1;occ=0;st=3;sb=3" tma_kernel
cap tma_t15 c5_t15 "kern=tma;kx=2;ky=1;tx=648;ty=2;order=1;occ=0;st=8;sb=3" tma_kernel
cap tma_t18 c5_t18 "kern=tma;kx=3;ky=1;tx=160;ty=36;order=0;occ=0;st=2;sb=2" tma_kernel
cap btile_t22 c5_t22 "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=2;bp=1;vec=3;ly=16" btile_kernel
cap btile_t14 c5_t14 "kern=smem;kx=1;ky=1;tx=64;ty=66;order=0;occ=0;st=2;bp=1;vec=3;ly=16" btile_kernel
cap rows_t04 c5_t04 "kern=copy;v=1;kx=0;ky=0;tx=1;ty=1;order=2;occ=0" copy_rows_kernel
cap rows_t19 c5_t19 "kern=copy;v=2;kx=0;ky=0;tx=1;ty=1;order=2;occ=0" copy_rows_kernel
cap vtile_c1 c1 "kern=smem;kx=1;ky=1;tx=64;ty=64;order=0;occ=0;st=2;bp=1;vec=1" vtile_kernel
cap copy_c2b c2b "kern=copy;v=4;kx=1;ky=1;tx=8;ty=8;order=0;occ=0" copy_kernel
ls gpurun_out/ | grep ncu_ | head -40
