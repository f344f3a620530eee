#!/bin/bash
for d in 0 1 2 3; do
  echo "debug=$d"
  MCKG_DEBUG=$d python bench.py --steps 10 --warmup 3 --no-cpu --no-k1 --e2e-blocks 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['config']['reported_triples'])"
done
