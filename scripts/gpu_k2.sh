#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_race.py tests/test_gpu_stuck.py -x -q > gpurun_out/k2tests.log 2>&1; echo "k2 tests rc=$?"
tail -15 gpurun_out/k2tests.log
for d in 0 1 2; do
  echo "debug=$d"
  MCKG_DEBUG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-k1 --e2e-blocks 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['config']['reported_triples'])"
done
