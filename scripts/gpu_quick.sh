#!/bin/bash
# parity corpus + full-size timing of the K1 path
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_programs.py -x -q > gpurun_out/prog.log 2>&1; echo "programs rc=$?"
tail -25 gpurun_out/prog.log
timeout 900 python scripts/gpu_fullsize.py ${FULL:-c2} > gpurun_out/full.log 2>&1; echo "full rc=$?"
cat gpurun_out/full.log
