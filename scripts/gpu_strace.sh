NQ_SHARD_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29871 bench.py --gpus 4 --steps 2 --warmup 3 --no-secondary > gpurun_out/strace.json 2> gpurun_out/strace.err; echo rc=$?
grep '\[shard\]' gpurun_out/strace.err | tail -40
