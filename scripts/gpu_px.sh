timeout 1500 python -m pytest tests/test_jit_gpu.py tests/test_sv_gpu.py tests/test_golden_gpu.py tests/test_dm_gpu.py -x -q > gpurun_out/px_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/px_pytest.log
for px in 1 0; do
NQ_JIT_PX=$px timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/px_$px.json 2> gpurun_out/px_$px.err; echo "px=$px rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['secondary']; print(d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], 'qft', s['qft30']['ms_per_circuit'], 'vqe', s['vqe28']['ms_per_eval'], 'dm14', s['dm_noisy_tfim14']['wall_s'], 'dm16', s['dm_noisy_tfim16']['wall_s'])" gpurun_out/px_$px.json
done
