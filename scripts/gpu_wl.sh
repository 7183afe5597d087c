timeout 1500 python -m pytest tests/test_jit_gpu.py tests/test_sv_gpu.py tests/test_golden_gpu.py tests/test_apps_gpu.py -x -q > gpurun_out/wl_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/wl_pytest.log
for wl in 1 0 1; do
NQ_JIT_WARPLOCAL=$wl timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/wl_$wl.json 2> gpurun_out/wl_$wl.err; echo "wl=$wl rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['secondary']; print(d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], 'qft', s['qft30']['ms_per_circuit'], 'vqe', s['vqe28']['ms_per_eval'], 'dm14', s['dm_noisy_tfim14']['wall_s'], 'qaoa', s['dm_noisy_qaoa14']['wall_s'])" gpurun_out/wl_$wl.json
done
