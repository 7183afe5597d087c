timeout 900 python -m pytest tests/test_dm_gpu.py -x -q > gpurun_out/c4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/c4_pytest.log
timeout 900 python bench.py > gpurun_out/c4_bench.json 2> gpurun_out/c4_bench.err; echo "bench rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['secondary']; print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value']); print({k:(v.get('wall_s') or v.get('ms_per_circuit') or v.get('ms_per_eval')) for k,v in s.items() if isinstance(v,dict)})" gpurun_out/c4_bench.json
