# column walk with precomputed byte offsets: parity, then A/B against the previous walk (whole sweep, alternating)
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tma.py tests/test_gpu_canary.py -q -x -m gpu -p no:cacheprovider > gpurun_out/walk_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/walk_tests.log
for i in 1 2; do
for v in new oldwalk; do
if [ $v = oldwalk ]; then export TTB_LIB_PATH=$PWD/paper_1603_02297_b200/_lib/libttb_oldwalk.so; else unset TTB_LIB_PATH; fi
timeout 900 python bench.py --no-cpu --no-e2e --no-configs > gpurun_out/walk_${v}_$i.json 2> gpurun_out/walk_${v}_$i.err; echo "$v $i rc=$?"
python - <<PY
import json
d=json.loads(open('gpurun_out/walk_${v}_$i.json').read().strip().splitlines()[-1])
print('$v', d['value'], d['pct_hbm_peak'], d['per_row_pass']['value'], d['clocks'], d['checksums_ok'])
print(' '.join(f"{r['row'][-3:]}={r['gbs']:.0f}" for r in d['rows']))
PY
done; done
