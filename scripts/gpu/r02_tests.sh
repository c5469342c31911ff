# full GPU suite, then the default bench
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"
tail -3 gpurun_out/bench_default.err
