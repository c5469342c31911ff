# TMA tile: separate A / B ring depths
for c in c1 c2a c3 c4 c5_t15 c5_t18 c5_t23 c5_t02 c5_t20 c5_t21 c5_t03; do
  timeout 300 python scripts/run_case.py $c --iters 8 --filter kern=tma \
    --extra "kern=tma;kx=1;ky=1;tx=32;ty=72;order=0;occ=0;st=8;sb=3" \
    --extra "kern=tma;kx=1;ky=1;tx=96;ty=24;order=0;occ=0;st=8;sb=3" \
    --extra "kern=tma;kx=1;ky=1;tx=64;ty=64;order=0;occ=0;st=6;sb=3" \
    --extra "kern=tma;kx=1;ky=1;tx=128;ty=32;order=0;occ=0;st=6;sb=3" \
    --extra "kern=tma;kx=1;ky=1;tx=32;ty=128;order=0;occ=0;st=6;sb=3" \
    --extra "kern=tma;kx=1;ky=1;tx=64;ty=64;order=0;occ=0;st=3;sb=2" \
    > gpurun_out/tma2_$c.log 2>&1
  head -1 gpurun_out/tma2_$c.log; grep -v "^#" gpurun_out/tma2_$c.log | sort -k3 -n -r | head -6
done
