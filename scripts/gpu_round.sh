#!/bin/bash
# One gpurun call: smoke, GPU tests, a bench line, the ncu launch list and one
# full ncu capture of the detector.  Outputs land in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
if [ -z "$NO_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-k1 --no-c5 --e2e-blocks 0 \
  > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fast_kernel|race_detect" -s 6 -c 2 \
  -o gpurun_out/prof_detect python bench.py --steps 3 --warmup 3 --no-cpu --no-k1 --no-c5 --e2e-blocks 0 \
  > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python scripts/ncu_summary.py gpurun_out/prof_detect.ncu-rep 25 > gpurun_out/k2_ncu_summary.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bucket|span|scan|tile" --csv \
  --log-file gpurun_out/c5_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-k1 --e2e-blocks 0 --blocks 1024 \
  > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
fi
