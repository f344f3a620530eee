#!/bin/bash
# compute-sanitizer memcheck + synccheck over a K2 and a K1 subset (one gpurun call).
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_race.py -q -x \
    -k "random_traces and (0 or 5 or 9) and two_kernel" > gpurun_out/san_k2_$tool.log 2>&1
  echo "K2 $tool rc=$?"; tail -1 gpurun_out/san_k2_$tool.log
  timeout 500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_gpu_programs.py -q -x \
    -k "fig1 or rich1 or conc1" > gpurun_out/san_k1_$tool.log 2>&1
  echo "K1 $tool rc=$?"; tail -1 gpurun_out/san_k1_$tool.log
done
