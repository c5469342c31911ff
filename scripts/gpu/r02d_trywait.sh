# A/B of the mbarrier wait: the product (mbarrier.try_wait, sleeping) against the spinning
# form (mbarrier.test_wait), whole sweep, alternating runs on one box.  Build the spinning
# library first (here, not on the GPU box):
#   python paper_1603_02297_b200/_build.py --variant spinwait TTB_SPIN_WAIT \
#       --only=kern_btile.cu --only=kern_btile_big.cu --only=kern_tma.cu --only=kern_rows.cu
# (profiles/r02_trywait_ab.log was taken when the spinning form was still the product.)
for i in 1 2; do
for v in product spinwait; do
if [ $v = spinwait ]; then export TTB_LIB_PATH=$PWD/paper_1603_02297_b200/_lib/libttb_spinwait.so; else unset TTB_LIB_PATH; fi
timeout 900 python bench.py --no-cpu --no-e2e --no-configs > gpurun_out/tw_${v}_$i.json 2> gpurun_out/tw_${v}_$i.err; echo "$v $i rc=$?"
python - <<PY
import json
d=json.loads(open('gpurun_out/tw_${v}_$i.json').read().strip().splitlines()[-1])
print('$v', d['value'], d['pct_hbm_peak'], d['per_row_pass']['value'], d['clocks'], d['checksums_ok'])
print([ (r['row'][-3:], r['gbs']) for r in d['rows']])
PY
done; done
