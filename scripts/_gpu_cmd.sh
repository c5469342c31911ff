S=$(date +%s); python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_secs=$(( $(date +%s) - S ))" >> gpurun_out/bench.err
S=$(date +%s); python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref_secs=$(( $(date +%s) - S ))" >> gpurun_out/bench_ref.err
