# A/B: prefetched tile claims; chunk walk (vec=5) on the slow rows, with checksums
run() { r=$1; shift; args=(); for p in "$@"; do args+=(--extra "$p"); done
  timeout 600 python scripts/run_case.py $r --filter NOCAND --iters 10 --check "${args[@]}" 2>&1 | tail -n +2; }
T14="kern=smem;kx=1;ky=1;tx=60;ty=197;order=0;occ=0;st=2;bp=1;vec=3;ts=1"
T14b="kern=smem;kx=1;ky=1;tx=28;ty=197;order=0;occ=0;st=2;bp=1;vec=3;ts=1"
T00="kern=smem;kx=2;ky=2;tx=128;ty=128;order=1;occ=0;st=2;bp=1;vec=3"
T13="kern=smem;kx=1;ky=1;tx=74;ty=64;order=0;occ=0;st=2;bp=1;vec=3"
for i in 1 2; do
echo "== prefetch on"; run c5_t14 "$T14" "$T14b"; run c5_t00 "$T00"; run c5_t13 "$T13"
echo "== prefetch off"; export TTB_NO_PREFETCH=1; run c5_t14 "$T14" "$T14b"; run c5_t00 "$T00"; run c5_t13 "$T13"; unset TTB_NO_PREFETCH
done
echo "== chunk walk t22"; run c5_t22 \
 "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=2;bp=1;vec=3;ly=16" \
 "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=2;bp=1;vec=5" \
 "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=2;bp=1;vec=5;ly=16" \
 "kern=smem;kx=1;ky=1;tx=71;ty=64;order=0;occ=0;st=2;bp=1;vec=5" \
 "kern=smem;kx=1;ky=1;tx=95;ty=128;order=0;occ=0;st=2;bp=1;vec=5" \
 "kern=smem;kx=1;ky=1;tx=95;ty=64;order=0;occ=0;st=2;bp=0;vec=5"
echo "== chunk walk t06"; run c5_t06 \
 "kern=smem;kx=2;ky=1;tx=128;ty=21;order=0;occ=0;st=2;bp=1;vec=3;ly=8" \
 "kern=smem;kx=2;ky=1;tx=128;ty=21;order=0;occ=0;st=2;bp=1;vec=5" \
 "kern=smem;kx=1;ky=1;tx=216;ty=21;order=0;occ=0;st=2;bp=1;vec=5" \
 "kern=smem;kx=1;ky=1;tx=108;ty=21;order=0;occ=0;st=2;bp=1;vec=5" \
 "kern=smem;kx=1;ky=1;tx=108;ty=21;order=0;occ=0;st=3;bp=1;vec=5"
echo "== chunk walk t14"; run c5_t14 \
 "kern=smem;kx=1;ky=1;tx=60;ty=197;order=0;occ=0;st=2;bp=1;vec=5;ts=1" \
 "kern=smem;kx=1;ky=1;tx=28;ty=197;order=0;occ=0;st=2;bp=1;vec=5;ts=1" \
 "kern=smem;kx=1;ky=1;tx=60;ty=66;order=0;occ=0;st=2;bp=1;vec=5;ts=1" \
 "kern=smem;kx=1;ky=1;tx=64;ty=66;order=0;occ=0;st=2;bp=1;vec=5"
echo "== chunk walk t00"; run c5_t00 \
 "kern=smem;kx=2;ky=2;tx=128;ty=128;order=1;occ=0;st=2;bp=1;vec=5" \
 "kern=smem;kx=2;ky=2;tx=64;ty=64;order=1;occ=0;st=2;bp=1;vec=5" \
 "kern=smem;kx=2;ky=2;tx=64;ty=64;order=1;occ=0;st=2;bp=1;vec=3"
echo "== chunk walk t07 (d) t13 (d, beta=0) t23"; run c5_t07 \
 "kern=smem;kx=1;ky=1;tx=32;ty=64;order=0;occ=0;st=2;bp=1;vec=3;ts=2" \
 "kern=smem;kx=1;ky=1;tx=32;ty=64;order=0;occ=0;st=2;bp=1;vec=5;ts=2" \
 "kern=smem;kx=1;ky=1;tx=32;ty=64;order=0;occ=0;st=2;bp=1;vec=5"
run c5_t13 "$T13" "kern=smem;kx=1;ky=1;tx=74;ty=64;order=0;occ=0;st=2;bp=1;vec=5"
run c5_t10 "kern=smem;kx=1;ky=2;tx=44;ty=2;order=0;occ=0;st=2;bp=1;vec=3" "kern=smem;kx=1;ky=2;tx=44;ty=2;order=0;occ=0;st=2;bp=1;vec=5"
