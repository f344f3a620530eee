#!/bin/bash
# ncu --set full of the K6 tile path (tile_claim + tile_mixed, one C5 call of 2^29 records)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tile_claim|tile_mixed" -c 2 \
  -o gpurun_out/prof_c5t env C5_REPS=1 C5_BLOCKS=131072 python scripts/c5_timing.py tile > gpurun_out/ncu_c5t.log 2>&1; echo "rc=$?"
for k in tile_claim tile_mixed; do
  echo "=== $k"; python scripts/ncu_summary.py gpurun_out/prof_c5t.ncu-rep 25 "$k" 2>&1
done > gpurun_out/c5t_summary.txt
