# explicit plans: whole-column tiles (B tile contiguous), deeper rings
run() { r=$1; shift; args=(); for p in "$@"; do args+=(--extra "$p"); done
  timeout 600 python scripts/run_case.py $r --top 1 --iters 8 --check "${args[@]}" 2>&1 | tail -n +2; }
echo "== t14"; run c5_t14 \
 "kern=smem;kx=1;ky=1;tx=60;ty=66;order=0;occ=0;st=2;bp=1;vec=3;ts=1" \
 "kern=smem;kx=1;ky=1;tx=60;ty=197;order=0;occ=0;st=2;bp=1;vec=3;ts=1" \
 "kern=smem;kx=1;ky=1;tx=28;ty=197;order=0;occ=0;st=2;bp=1;vec=3;ts=1" \
 "kern=smem;kx=1;ky=1;tx=28;ty=197;order=0;occ=0;st=3;bp=1;vec=3;ts=1" \
 "kern=smem;kx=1;ky=1;tx=60;ty=197;order=0;occ=0;st=2;bp=1;vec=4;ts=1" \
 "kern=smem;kx=1;ky=1;tx=28;ty=197;order=0;occ=0;st=3;bp=1;vec=4;ts=1" \
 "kern=smem;kx=1;ky=1;tx=60;ty=197;order=0;occ=0;st=2;bp=1;vec=3" \
 "kern=smem;kx=1;ky=1;tx=64;ty=197;order=0;occ=0;st=2;bp=1;vec=4" \
 "kern=smem;kx=1;ky=1;tx=32;ty=197;order=0;occ=0;st=3;bp=1;vec=4"
echo "== t06"; run c5_t06 \
 "kern=smem;kx=2;ky=1;tx=128;ty=21;order=0;occ=0;st=2;bp=1;vec=3;ly=8" \
 "kern=smem;kx=1;ky=1;tx=216;ty=21;order=0;occ=0;st=2;bp=1;vec=3;ly=8" \
 "kern=smem;kx=1;ky=1;tx=216;ty=21;order=0;occ=0;st=3;bp=1;vec=3;ly=8" \
 "kern=smem;kx=1;ky=1;tx=216;ty=21;order=0;occ=0;st=4;bp=1;vec=3;ly=8" \
 "kern=smem;kx=1;ky=1;tx=216;ty=21;order=0;occ=0;st=2;bp=1;vec=3;ly=8;ts=1" \
 "kern=smem;kx=1;ky=1;tx=216;ty=21;order=0;occ=0;st=3;bp=1;vec=4" \
 "kern=smem;kx=1;ky=1;tx=216;ty=21;order=0;occ=0;st=2;bp=0;vec=3;ly=8"
echo "== t00"; run c5_t00 \
 "kern=smem;kx=2;ky=2;tx=128;ty=128;order=1;occ=0;st=2;bp=1;vec=3" \
 "kern=smem;kx=2;ky=2;tx=128;ty=96;order=1;occ=0;st=3;bp=1;vec=3" \
 "kern=smem;kx=2;ky=2;tx=96;ty=128;order=1;occ=0;st=3;bp=1;vec=3" \
 "kern=smem;kx=2;ky=2;tx=128;ty=64;order=1;occ=0;st=4;bp=1;vec=3" \
 "kern=smem;kx=2;ky=2;tx=256;ty=64;order=1;occ=0;st=2;bp=1;vec=3" \
 "kern=smem;kx=2;ky=2;tx=256;ty=48;order=1;occ=0;st=3;bp=1;vec=3"
echo "== t22"; run c5_t22 \
 "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=2;bp=1;vec=3;ly=16" \
 "kern=smem;kx=1;ky=1;tx=283;ty=32;order=0;occ=0;st=2;bp=1;vec=3" \
 "kern=smem;kx=1;ky=1;tx=283;ty=64;order=0;occ=0;st=2;bp=1;vec=3" \
 "kern=smem;kx=1;ky=1;tx=283;ty=16;order=0;occ=0;st=3;bp=1;vec=3" \
 "kern=smem;kx=1;ky=1;tx=142;ty=128;order=0;occ=0;st=2;bp=1;vec=3" \
 "kern=smem;kx=1;ky=1;tx=95;ty=128;order=0;occ=0;st=2;bp=1;vec=3" \
 "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=3;bp=1;vec=3;ly=16" \
 "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=4;bp=1;vec=3;ly=16"
cap() {  # name case plan kernel-regex
  python scripts/run_case.py $2 --plan "$3" --iters 2 > gpurun_out/ncu_$1_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$4 -s 1 -c 1 -o /tmp/ncu_$1 \
      python scripts/run_case.py $2 --plan "$3" --iters 2 > gpurun_out/ncu_$1.log 2>&1 && \
  ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv && \
  ncu -i /tmp/ncu_$1.ncu-rep --page source --csv > gpurun_out/ncu_$1_source.csv
  echo "$1 rc=$?"; rm -f /tmp/ncu_$1.ncu-rep
}
cap btile_t06 c5_t06 "kern=smem;kx=1;ky=1;tx=216;ty=21;order=0;occ=0;st=2;bp=1;vec=3;ly=8" btile_kernel
