NQ_BENCH_LAPS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 5 --warmup 3 --no-secondary > gpurun_out/bench_n2l.json 2> gpurun_out/bench_n2l.err; echo "rc=$?"
grep 'e2e step' gpurun_out/bench_n2l.err
python -c "import json; d=json.loads(open('gpurun_out/bench_n2l.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
