W=${W:-4}
timeout 900 python -m pytest tests/test_shard_gpu.py -x -q > gpurun_out/n4_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/n4_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $W > gpurun_out/n${W}_bench.json 2> gpurun_out/n${W}_bench.err; echo "bench rc=$?"
cat gpurun_out/n${W}_bench.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $W --impl reference > gpurun_out/n${W}_ref.json 2> gpurun_out/n${W}_ref.err; echo "ref rc=$?"
cat gpurun_out/n${W}_ref.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 > gpurun_out/n2_bench.json 2> gpurun_out/n2_bench.err; echo "bench2 rc=$?"
cat gpurun_out/n2_bench.json
