set -x
W=${W:-2}
timeout 900 python -m pytest tests/test_shard_gpu.py -x -q > gpurun_out/fx_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/fx_pytest.log
for fx in 1 0; do
export NQ_BENCH_LAPS=1
NQ_FUSED_EXCHANGE=$fx timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $W --steps 10 --warmup 3 > gpurun_out/fx_bench_w${W}_f$fx.json 2> gpurun_out/fx_bench_w${W}_f$fx.err; echo "bench fx=$fx rc=$?"
cat gpurun_out/fx_bench_w${W}_f$fx.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["passes_per_step"], d["config"]["comm"], d["roofline"]["avg_launch_ms"], d["e2e"]["value"])"
done
NQ_SHARD_TRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29512 scripts/shard_probe.py > gpurun_out/fx_probe_w$W.log 2>&1; echo "probe rc=$?"
grep -v "^\[shard\] segment" gpurun_out/fx_probe_w$W.log | tail -20
