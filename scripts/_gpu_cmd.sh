for p in "tx=16;ty=197;order=0;occ=0;st=2;bp=1;vec=1" "tx=16;ty=197;order=0;occ=0;st=2;bp=0;vec=1" "tx=16;ty=197;order=0;occ=0;st=2;bp=1;vec=0" "tx=16;ty=197;order=0;occ=0;st=2;bp=0;vec=0" "tx=32;ty=197;order=0;occ=0;st=2;bp=1;vec=1" "tx=32;ty=197;order=0;occ=0;st=2;bp=0;vec=1" "tx=8;ty=197;order=0;occ=0;st=2;bp=1;vec=1" "tx=8;ty=197;order=0;occ=0;st=2;bp=0;vec=0" "tx=64;ty=99;order=0;occ=0;st=2;bp=0;vec=1" "tx=128;ty=66;order=0;occ=0;st=2;bp=0;vec=1"; do
python scripts/run_case.py c5_t14 --iters 5 --plan "kern=smem;kx=1;ky=1;$p" | tail -1
done > gpurun_out/t14.log 2>&1
