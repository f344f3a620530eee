for d in 2 9 17 1 0; do
  echo "debug=$d $(MCKG_DEBUG=$d python bench.py --steps 10 --warmup 3 --no-cpu --no-k1 --no-c5 --e2e-blocks 0 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["roofline"]["kernel_ms"])')"
done
