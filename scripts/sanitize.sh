#!/bin/bash
# compute-sanitizer (memcheck, synccheck, racecheck) over small cases of every
# kernel family, one gpurun call: K2 fast + general, K6 tile path + bucket
# pipeline, K1 (whole programs incl. serial tails), K7 oracle.
mkdir -p gpurun_out
run() {  # tool name pytest-args...
  local tool=$1 name=$2; shift 2
  timeout 600 compute-sanitizer --tool $tool --print-limit 5 python -m pytest -q -x "$@" \
    > gpurun_out/san_${name}_$tool.log 2>&1
  echo "$name $tool rc=$? $(grep -h 'ERROR SUMMARY' gpurun_out/san_${name}_$tool.log | sort | uniq -c | tr '\n' ' ')"
}
for tool in memcheck synccheck racecheck; do
  run $tool k2 tests/test_gpu_race.py -k "random_traces and (0 or 5) or hot_word or hands_back"
  run $tool k6 tests/test_gpu_global.py -k "c5_sample or block_clustered or random_global_traces and 0"
  run $tool k1 tests/test_gpu_programs.py -k "fig1 or rich_random_programs and (1 or 2) or divergent"
  run $tool k7 tests/test_gpu_oracle.py -k "matches_reference"
done
