#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bucket_fast|bucket_scatter|bucket_count" -c 3 \
  -o gpurun_out/prof_c5 python bench.py --steps 1 --warmup 3 --no-cpu --no-k1 --e2e-blocks 0 --blocks 1024 \
  > gpurun_out/ncu_c5.log 2>&1; echo "rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_c5.ncu-rep 25 > gpurun_out/c5_summary.txt 2>&1
