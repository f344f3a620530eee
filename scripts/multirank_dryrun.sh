# functional dry run of the multi-rank bench on one GPU (gloo, all ranks on cuda:0)
for n in 2 4; do
MCKG_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29$((500+n)) \
  bench.py --gpus $n --steps 3 --warmup 3 --blocks 65536 --c5-blocks 4096 > gpurun_out/mr$n.json 2> gpurun_out/mr$n.err; echo "n=$n rc=$?"
python -c "import json; d=json.load(open('gpurun_out/mr$n.json')); print(d['n_gpus'], d['value'], d['config']['reported_triples'], d['c5'])"
tail -2 gpurun_out/mr$n.err
done
