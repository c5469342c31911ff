for s in 1 2 3 4; do
timeout 900 python bench.py --streams $s --no-cpu --no-e2e --no-configs > gpurun_out/streams_$s.json 2> gpurun_out/streams_$s.err; echo "streams $s rc=$?"
python - <<PY
import json
d=json.loads(open('gpurun_out/streams_$s.json').read().strip().splitlines()[-1])
print($s, d['value'], d['pct_hbm_peak'], d['pct_d2d'], d['one_stream'], d['clocks'], d['checksums_ok'], d['gpu_launches'])
PY
done
