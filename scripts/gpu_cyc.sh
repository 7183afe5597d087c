timeout 600 python -m pytest tests/test_shard_gpu.py -x -q 2>&1 | tail -1
for cfg in "4 30 1" "4 30 0" "4 33 1" "2 30 1"; do
set -- $cfg
NQ_SHARD_CYCLIC=$3 timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 298$1$3 bench.py --gpus $1 --qubits $2 --steps 5 --warmup 3 --no-secondary > gpurun_out/cyc_$1_$2_$3.json 2> gpurun_out/cyc_$1_$2_$3.err; echo "N=$1 local=$2 cyclic=$3 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/cyc_$1_$2_$3.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['passes_per_step'], d['config']['comm'], d['e2e']['value'])"
done
