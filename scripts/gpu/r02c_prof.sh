# where the time goes on the slow bulk-tile rows: beta overrides, then ncu --set full with the source page
for r in c5_t22 c5_t14 c5_t06; do
  timeout 600 python scripts/run_case.py $r --beta 0 --filter "vec=3" --top 12 --iters 8 > gpurun_out/beta0_$r.log 2>&1
  echo "$r beta0 rc=$?"; sort -k3 -n -r gpurun_out/beta0_$r.log | head -4
done
timeout 600 python scripts/run_case.py c5_t00 --beta 0.5 --filter "vec=3" --top 12 --iters 8 > gpurun_out/beta5_c5_t00.log 2>&1
sort -k3 -n -r gpurun_out/beta5_c5_t00.log | head -4
cap() {  # name case plan kernel-regex
  python scripts/run_case.py $2 --plan "$3" --iters 2 > gpurun_out/ncu_$1_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 -o /tmp/ncu_$1 \
      python scripts/run_case.py $2 --plan "$3" --iters 2 > gpurun_out/ncu_$1.log 2>&1 && \
  ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv && \
  ncu -i /tmp/ncu_$1.ncu-rep --page source --csv > gpurun_out/ncu_$1_source.csv
  echo "$1 rc=$?"; rm -f /tmp/ncu_$1.ncu-rep
}
cap btile_t14 c5_t14 "kern=smem;kx=1;ky=1;tx=60;ty=66;order=0;occ=0;st=2;bp=1;vec=3;ts=1" btile_kernel
cap btile_t22 c5_t22 "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=2;bp=1;vec=3;ly=16" btile_kernel
cap btile_t00 c5_t00 "kern=smem;kx=2;ky=2;tx=128;ty=128;order=1;occ=0;st=2;bp=1;vec=3" btile_kernel
ls -la gpurun_out | head -40
