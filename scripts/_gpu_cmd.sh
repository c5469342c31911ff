for lib in libttb.so libttb_mb1.so libttb_mb4.so; do
for cv in -1 50; do
for c in c5_t00 c5_t16 c5_t22; do
  echo "== lib=$lib cv=$cv"
  TTB_LIB_PATH=$PWD/paper_1603_02297_b200/_lib/$lib TTB_CARVEOUT=$cv timeout 200 python scripts/run_case.py $c --iters 5 --top 8
done; done; done > gpurun_out/var.log 2>&1
