timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
