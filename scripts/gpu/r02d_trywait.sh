# A/B: mbarrier.test_wait spin (product) vs mbarrier.try_wait, whole sweep, alternating
for i in 1 2; do
for v in product trywait; do
if [ $v = trywait ]; then export TTB_LIB_PATH=$PWD/paper_1603_02297_b200/_lib/libttb_trywait.so; else unset TTB_LIB_PATH; fi
timeout 900 python bench.py --no-cpu --no-e2e --no-configs > gpurun_out/tw_${v}_$i.json 2> gpurun_out/tw_${v}_$i.err; echo "$v $i rc=$?"
python - <<PY
import json
d=json.loads(open('gpurun_out/tw_${v}_$i.json').read().strip().splitlines()[-1])
print('$v', d['value'], d['pct_hbm_peak'], d['per_row_pass']['value'], d['clocks'], d['checksums_ok'])
print([ (r['row'][-3:], r['gbs']) for r in d['rows']])
PY
done; done
