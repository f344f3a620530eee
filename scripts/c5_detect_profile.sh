#!/bin/bash
# ncu --set full of K6's bucket_fast_kernel alone (one C5 call)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bucket_fast" -c 1 \
  -o gpurun_out/prof_c5d python bench.py --steps 1 --warmup 3 --no-cpu --no-k1 --e2e-blocks 0 --blocks 1024 \
  > gpurun_out/ncu_c5d.log 2>&1; echo "rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_c5d.ncu-rep 30 > gpurun_out/c5d_summary.txt 2>&1
