#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel|race_detect" -s 2 -c 2 \
  -o gpurun_out/prof_k2_fast python bench.py --steps 2 --warmup 3 --no-cpu --no-k1 --no-c5 --e2e-blocks 0 \
  > gpurun_out/ncu_k2fast.log 2>&1; echo "rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_k2_fast.ncu-rep 30 > gpurun_out/k2_fast_summary.txt 2>&1
