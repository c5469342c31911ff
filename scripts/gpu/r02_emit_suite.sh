timeout 1200 python -m pytest tests/test_gpu_emit.py tests/test_gpu_suite.py tests/test_cli.py "tests/test_gpu_parity.py::test_tune_cached_miss_then_hit" -q -p no:cacheprovider > gpurun_out/emit_suite_tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/emit_suite_tests.log
timeout 1500 python scripts/suite.py --ref --verify --csv gpurun_out/r02_suite_200MiB_s.csv > gpurun_out/r02_suite_200MiB_s.log 2>&1
echo "suite rc=$?"; tail -5 gpurun_out/r02_suite_200MiB_s.log
