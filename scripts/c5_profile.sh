#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 400 --csv \
  --log-file gpurun_out/c5_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-k1 --e2e-blocks 0 --blocks 1024 > gpurun_out/c5_ncu.log 2>&1; echo "rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/c5_launches.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r))
        print(d['ID'], d['Kernel Name'][:40], d['Metric Name'], d['Metric Value'])
PY
