# probe: the big warp roles (8 consumer + 4 producer warps) on tiles below 32 KB
run() { r=$1; shift; args=(); for p in "$@"; do args+=(--extra "$p"); done
  timeout 600 python scripts/run_case.py $r --filter NOCAND --iters 10 --check "${args[@]}" 2>&1 | tail -n +2; }
for bb in 32768 8192 16384; do
export TTB_BIG_BYTES=$bb; echo "== big roles from $bb bytes"
run c5_t22 "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=2;bp=1;vec=3;ly=16" "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=2;bp=1;vec=3" "kern=smem;kx=1;ky=1;tx=71;ty=64;order=0;occ=0;st=2;bp=1;vec=3;ly=16"
run c5_t06 "kern=smem;kx=2;ky=1;tx=128;ty=21;order=0;occ=0;st=2;bp=1;vec=3;ly=8" "kern=smem;kx=1;ky=1;tx=216;ty=21;order=0;occ=0;st=2;bp=1;vec=3;ly=8" "kern=smem;kx=1;ky=1;tx=108;ty=21;order=0;occ=0;st=2;bp=1;vec=3;ly=8"
run c5_t14 "kern=smem;kx=1;ky=1;tx=60;ty=66;order=0;occ=0;st=2;bp=1;vec=3;ts=1" "kern=smem;kx=1;ky=1;tx=28;ty=197;order=0;occ=0;st=2;bp=1;vec=3;ts=1"
run c5_t00 "kern=smem;kx=2;ky=2;tx=64;ty=64;order=1;occ=0;st=2;bp=1;vec=3" "kern=smem;kx=1;ky=1;tx=79;ty=82;order=0;occ=0;st=2;bp=1;vec=3"
run c5_t07 "kern=smem;kx=1;ky=1;tx=32;ty=64;order=0;occ=0;st=2;bp=1;vec=3;ts=2"
run c5_t13 "kern=smem;kx=1;ky=1;tx=74;ty=64;order=0;occ=0;st=2;bp=1;vec=3"
run c5_t09 "kern=smem;kx=2;ky=1;tx=64;ty=75;order=1;occ=0;st=2;bp=1;vec=3"
done
