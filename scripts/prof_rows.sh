# ncu --set full of one launch per (row, plan) -- kernel-design probe.
# usage: bash scripts/prof_rows.sh ROW "PLAN" [ROW "PLAN" ...]
# Reports stay in /tmp/prof (too large to bring back); gpurun_out/ gets the
# summary (scripts/ncu_summary.py), the details page and the raw csv.
mkdir -p /tmp/prof
while [ $# -ge 2 ]; do
  row=$1; plan=$2; shift 2
  timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:'^(btile|dense|vtile|tile|copy|copy_rows|rt|smem)_kernel' -c 1 -f \
    -o /tmp/prof/prof_$row python scripts/run_case.py $row --plan "$plan" --iters 1 \
    > gpurun_out/prof_$row.log 2>&1
  echo "$row rc=$?" >> gpurun_out/prof_rows.log
  python scripts/ncu_summary.py /tmp/prof/prof_$row.ncu-rep > gpurun_out/prof_$row.summary.json 2>&1
  ncu -i /tmp/prof/prof_$row.ncu-rep --page details --csv > gpurun_out/prof_$row.details.csv 2>&1
  ncu -i /tmp/prof/prof_$row.ncu-rep --page raw --csv > gpurun_out/prof_$row.raw.csv 2>&1
done
