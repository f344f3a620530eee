for d in 2 1 0; do
  echo "== debug=$d"
  MCKG_DEBUG=$d timeout 120 python bench.py --steps 3 --warmup 3 --no-cpu --no-k1 --e2e-blocks 0 --blocks 4096 2>&1 | tail -2 | cut -c1-300
done
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_race.py -x -q -k "single_thread or hot_word" 2>&1 | grep -v "^\s*$" | head -20
