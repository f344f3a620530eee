#!/bin/bash
# compute-sanitizer synccheck + racecheck of K1 alone
mkdir -p gpurun_out
for tool in synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 5 python -m pytest -q -x tests/test_gpu_programs.py \
    -k "fig1 or rich_random_programs and (1 or 2) or divergent" > gpurun_out/san_k1_$tool.log 2>&1
  echo "k1 $tool rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' gpurun_out/san_k1_$tool.log | tr '\n' ' ')"
done
