#!/bin/bash
# ncu --set full (with source) of the K2 filter alone and of the whole
# detect call (filter + exact_kernel), C3 full size; reports in gpurun_out/.
mkdir -p gpurun_out
MCKG_DEBUG=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:race_detect -s 2 -c 1 \
  -o gpurun_out/prof_k2_filter python bench.py --steps 3 --warmup 3 --no-cpu --no-k1 --no-c5 --e2e-blocks 0 \
  > gpurun_out/ncu_k2f.log 2>&1; echo "filter rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"race_detect|exact_kernel" -s 6 -c 2 \
  -o gpurun_out/prof_k2_call python bench.py --steps 3 --warmup 3 --no-cpu --no-k1 --no-c5 --e2e-blocks 0 \
  > gpurun_out/ncu_k2c.log 2>&1; echo "call rc=$?"
