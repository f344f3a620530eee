#!/bin/bash
# ncu --set full of the K6 side-list bucket_fast (tile path, one C5 call)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bucket_fast" -c 1 \
  -o gpurun_out/prof_c5s env C5_REPS=1 python scripts/c5_timing.py tile > gpurun_out/ncu_c5s.log 2>&1; echo "rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_c5s.ncu-rep 30 > gpurun_out/c5s_summary.txt 2>&1
