timeout 2400 python scripts/predict_scaling.py --worlds 1,2,4,8 > gpurun_out/r02_predict_scaling.log 2>&1; echo "rc=$?"
grep world gpurun_out/r02_predict_scaling.log
timeout 1200 python -m pytest tests/test_gpu_shard_rows.py "tests/test_gpu_parity.py::test_sharded_execution_equals_single_call" -q -p no:cacheprovider 2>&1 | tail -2
