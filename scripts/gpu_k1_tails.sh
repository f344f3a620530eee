#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_programs.py tests/test_gpu_edge.py tests/test_gpu_trace.py -x -q > gpurun_out/k1_tail_tests.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/k1_tail_tests.log
timeout 300 python scripts/k1_timing.py 2>&1 | grep "{"
MCKG_K1_TAILS=0 timeout 300 python scripts/k1_timing.py 2>&1 | grep "{"
