timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-k1 --e2e-blocks 0 --blocks 4096 > /dev/null 2>&1; echo rc=$?
