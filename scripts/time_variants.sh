#!/bin/bash
# C3 timing of each build/variants/<name>/libmckg.so (plus the in-tree lib).
mkdir -p gpurun_out
for v in default $(ls build/variants); do
  lib=paper_1211_6193_b200/libmckg.so; [ "$v" != default ] && lib=build/variants/$v/libmckg.so
  MCKG_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-k1 --no-c5 --e2e-blocks 0 > gpurun_out/var_$v.json 2>&1
  echo "$v rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/var_$v.json').read().splitlines()[-1]); print(d['roofline']['kernel_ms'], round(d['roofline']['frac'],4), d['config']['reported_triples'])" 2>&1 | tail -1)"
done
