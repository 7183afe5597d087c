W=${W:-2}
export NQ_BENCH_LAPS=1 NQ_SHARD_TIMING=30
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $W --steps 10 --warmup 3 > gpurun_out/spike_w${W}.json 2> gpurun_out/spike_w${W}.err; echo "bench rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['passes_per_step'], d['config']['comm'], d['e2e'], d['jit'], d['jit_end'])" gpurun_out/spike_w${W}.json
grep -v "^\[shard\] segment" gpurun_out/spike_w${W}.err | grep "rank 0\|e2e" | tail -60
