# reference arm, engine arm, 2 ranks sharing the GPU (gloo), launch list of the timed region
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; echo "ref rc=$?"
timeout 1200 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
timeout 1200 python bench.py --gpus 2 --steps 3 --no-configs --no-cpu --no-e2e > gpurun_out/r02_bench_2rank_gloo.json 2> gpurun_out/r02_bench_2rank_gloo.err; echo "2rank rc=$?"
timeout 900 python bench.py --steps 1 --no-configs --no-cpu --no-e2e > gpurun_out/r02_launch_plain.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "ttb_timed/" --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --no-configs --no-cpu --no-e2e > gpurun_out/r02_launch_ncu.log 2>&1; echo "ncu rc=$?"
