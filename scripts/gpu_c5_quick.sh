#!/bin/bash
# K6 parity tests + a C5 timing line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_global.py -x -q > gpurun_out/c5_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/c5_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-k1 --e2e-blocks 0 --blocks 4096 > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err
echo "bench rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/c5_bench.json').read().splitlines()[-1])['c5']; print(d['ms_per_step'], d['roofline']['frac'], d['races_reported'], d['status'])" 2>&1 | tail -1)"
