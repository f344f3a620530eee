cp paper_1211_6193_b200/libmckg.so /tmp/libmckg.orig.so
for f in variants/libmckg_*.so; do
  cp $f paper_1211_6193_b200/libmckg.so
  echo "$f: $(python bench.py --steps 10 --warmup 3 --no-cpu --no-k1 --no-c5 --e2e-blocks 0 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["roofline"]["kernel_ms"], d["roofline"]["frac"], d["config"]["reported_triples"])')"
done
cp /tmp/libmckg.orig.so paper_1211_6193_b200/libmckg.so
