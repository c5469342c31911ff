timeout 1200 python -m pytest tests/test_gpu_tma.py -q -p no:cacheprovider -x > gpurun_out/diag_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/diag_tests.log
for c in c3 c5_t18 c5_t15 c5_t02 c5_t03 c1 c2a c4; do
  timeout 300 python scripts/run_case.py $c --iters 8 --filter kern=tma > gpurun_out/diag_$c.log 2>&1
  head -1 gpurun_out/diag_$c.log | cut -c1-50; grep -v "^#" gpurun_out/diag_$c.log | sort -k3 -n -r | head -2
done
P="kern=tma;kx=3;ky=1;tx=160;ty=36;order=0;occ=0;st=2;sb=2"
python scripts/run_case.py c5_t18 --plan "$P" --iters 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none -k regex:tma_kernel -s 1 -c 1 -o /tmp/ncu_diag python scripts/run_case.py c5_t18 --plan "$P" --iters 2 > /dev/null 2>&1 && \
ncu -i /tmp/ncu_diag.ncu-rep --page raw --csv > gpurun_out/ncu_tma_t18_diag_raw.csv; echo "ncu rc=$?"
