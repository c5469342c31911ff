# round-2 re-entry: full GPU suite and the default bench at HEAD
timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r02b_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['pct_hbm_peak'], d['pct_d2d'], d['clocks'], d.get('cpu_baseline',{}).get('value'))
print([(r['row'][-3:], r['gbs'], r['plan'].split('fn=')[-1]) for r in d['rows']])
print({k:(v['gbs'] if isinstance(v,dict) else v) for k,v in d['configs'].items()})
PY
