set -x
timeout 600 python -m pytest tests/test_shard_gpu.py -x -q > gpurun_out/pytest_shard.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_shard.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench$N rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_n$N.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['passes_per_step'], d['config']['comm'], d['e2e']['value'])"; tail -3 gpurun_out/bench_n$N.err
done
NQ_EXCHANGE=nccl timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29599 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_n4nccl.json 2> gpurun_out/bench_n4nccl.err; echo "bench4nccl rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_n4nccl.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['passes_per_step'], d['config']['comm'])"
