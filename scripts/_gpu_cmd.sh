timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" > gpurun_out/pytest_host.log 2>&1; echo rc=$? >> gpurun_out/pytest_host.log
timeout 600 python scripts/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; echo rc=$? >> gpurun_out/e2e_probe.log
