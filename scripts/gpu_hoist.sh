timeout 600 python -m pytest tests/test_shard_gpu.py -x -q 2>&1 | tail -1
for N in 4 2; do
for h in 1 0; do
NQ_SHARD_HOIST=$h timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 297$N$h bench.py --gpus $N --steps 5 --warmup 3 --no-secondary > gpurun_out/bench_n${N}_h$h.json 2> gpurun_out/bench_n${N}_h$h.err; echo "bench$N hoist=$h rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_n${N}_h$h.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['passes_per_step'], d['config']['comm'], d['e2e']['value'])"
done
done
