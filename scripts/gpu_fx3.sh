set -x
W=${W:-4}
timeout 900 python -m pytest tests/test_shard_gpu.py -x -q > gpurun_out/fx_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/fx_pytest.log
export NQ_BENCH_LAPS=1
for cfg in "1 1" "1 0"; do
set -- $cfg
NQ_FUSED_EXCHANGE=$1 NQ_SHARD_REBALANCE=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $W --steps 10 --warmup 3 > gpurun_out/fx_bench_w${W}_f$1_r$2.json 2> gpurun_out/fx_bench_w${W}_f$1_r$2.err; echo "bench $cfg rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['passes_per_step'], d['config']['comm'], d['roofline']['avg_launch_ms'], d['e2e'], d['jit'], d['jit_end'])" gpurun_out/fx_bench_w${W}_f$1_r$2.json
grep "e2e step" gpurun_out/fx_bench_w${W}_f$1_r$2.err | head -2
done
