#!/bin/bash
# K1 edge/capacity tests + C2/C4 timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edge.py -x -q > gpurun_out/k1_edge.log 2>&1; echo "edge rc=$?"; tail -5 gpurun_out/k1_edge.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-c5 --e2e-blocks 0 --blocks 1024 > gpurun_out/k1_bench.json 2> gpurun_out/k1_bench.err
echo "bench rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/k1_bench.json').read().splitlines()[-1])['k1']; print('C2', d['thread_steps_per_s'], d['grid_ms'], d['output_ok'], 'C4', d['c4']['thread_steps_per_s'], d['c4']['grid_ms'], d['c4']['deadlocks_ok'])" 2>&1 | tail -1)"
