set -x
nvidia-smi --query-gpu=index,name --format=csv
timeout 600 python -m pytest tests/test_shard_gpu.py -x -q > gpurun_out/pytest_shard.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_shard.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench$N rc=$?"
cat gpurun_out/bench_n$N.json; tail -5 gpurun_out/bench_n$N.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/bench_ref_n4.json 2> gpurun_out/bench_ref_n4.err; echo "ref4 rc=$?"
cat gpurun_out/bench_ref_n4.json; tail -5 gpurun_out/bench_ref_n4.err
