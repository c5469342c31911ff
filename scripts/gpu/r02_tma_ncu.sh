# ncu of the TMA tile on c2a (beta = 0) and a stage sweep
P="kern=tma;kx=1;ky=1;tx=96;ty=72;order=0;occ=0;st=3"
for st in 2 3 4 5 6; do
  python scripts/run_case.py c2a --plan "kern=tma;kx=1;ky=1;tx=96;ty=36;order=0;occ=0;st=$st" --iters 10 | tail -1
  python scripts/run_case.py c2a --plan "kern=tma;kx=1;ky=1;tx=48;ty=72;order=0;occ=0;st=$st" --iters 10 | tail -1
done
for t in "tx=32;ty=64" "tx=64;ty=32" "tx=64;ty=64" "tx=96;ty=24" "tx=32;ty=72" "tx=96;ty=48"; do
  for st in 3 4 6; do
  python scripts/run_case.py c2a --plan "kern=tma;kx=1;ky=1;$t;order=0;occ=0;st=$st" --iters 10 | tail -1
  done
done
python scripts/run_case.py c2a --plan "$P" --iters 3 > gpurun_out/c2a_tma_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tma_kernel -s 2 -c 1 -o /tmp/c2a_tma python scripts/run_case.py c2a --plan "$P" --iters 3 > gpurun_out/c2a_tma_ncu.log 2>&1
ncu -i /tmp/c2a_tma.ncu-rep --page raw --csv > gpurun_out/c2a_tma_raw.csv
ncu -i /tmp/c2a_tma.ncu-rep --page details --csv > gpurun_out/c2a_tma_details.csv
ncu -i /tmp/c2a_tma.ncu-rep --page source --csv > gpurun_out/c2a_tma_source.csv 2>&1
ls -la gpurun_out
