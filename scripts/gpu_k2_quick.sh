#!/bin/bash
# K2 parity tests + a C3 timing line (no K1 / C5 / CPU legs).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_race.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/k2_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/k2_tests.log
for d in ${DEBUGS:-0}; do
  MCKG_DEBUG=$d timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-k1 --no-c5 --e2e-blocks 0 > gpurun_out/k2_bench_$d.json 2> gpurun_out/k2_bench_$d.err
  echo "debug=$d rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/k2_bench_$d.json').read().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['config']['reported_triples'])" 2>&1 | tail -1)"
done
