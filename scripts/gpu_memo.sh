timeout 1500 python -m pytest tests/test_sv_gpu.py tests/test_jit_gpu.py tests/test_shard_gpu.py tests/test_golden_gpu.py -x -q > gpurun_out/memo_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/memo_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/memo_n1.json 2> gpurun_out/memo_n1.err; echo "n1 rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['secondary']; print(d['value'], d['ms_per_step'], d['e2e'], 'vqe', s['vqe28']['ms_per_eval'], 'qft', s['qft30']['ms_per_circuit'])" gpurun_out/memo_n1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 > gpurun_out/memo_n2.json 2> gpurun_out/memo_n2.err; echo "n2 rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'])" gpurun_out/memo_n2.json
