#!/bin/bash
# ncu launch list (time, DRAM bytes) of one tile-path and one bucket-path C5 call
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c5_launch_list.csv python scripts/c5_timing.py tile buckets > gpurun_out/c5_launch.log 2>&1; echo "rc=$?"
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/c5_launch_list.csv')))
h = None
agg = {}
for r in rows:
    if r and r[0] == 'ID': h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        agg.setdefault(d['ID'], [d['Kernel Name'][:44], 0, 0, 0])
        k = {'gpu__time_duration.sum': 1, 'dram__bytes_read.sum': 2, 'dram__bytes_write.sum': 3}[d['Metric Name']]
        agg[d['ID']][k] = float(d['Metric Value'].replace(',', ''))
for i, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: int(x[0])):
    if 'at::' in n or 'gen_c5' in n: continue
    print(f"{i:>4} {n:44s} {t/1e3:9.1f} us  rd {rd/1e9:7.3f} GB  wr {wr/1e9:7.3f} GB")
PY
