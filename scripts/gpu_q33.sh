timeout 900 python bench.py --qubits 33 --steps 4 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/q33_n1.json 2> gpurun_out/q33_n1.err; echo "n1 rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['passes_per_step'], d['roofline']['frac'])" gpurun_out/q33_n1.json
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --qubits 33 --steps 4 --warmup 3 > gpurun_out/q33_n4.json 2> gpurun_out/q33_n4.err; echo "n4 rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['passes_per_step'], d['config']['comm'], d['roofline']['frac'], d['e2e']['value'])" gpurun_out/q33_n4.json
tail -3 gpurun_out/q33_n4.err
