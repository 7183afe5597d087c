set -x
nvidia-smi --query-gpu=index,name --format=csv
timeout 600 python -m pytest tests/test_shard_gpu.py -x -q > gpurun_out/pytest_shard.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_shard.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench2 rc=$?"
cat gpurun_out/bench_n2.json; tail -20 gpurun_out/bench_n2.err
