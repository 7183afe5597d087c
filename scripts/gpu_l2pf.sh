for pf in 0 1 2 0 1; do
NQ_JIT_L2PF=$pf timeout 600 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/l2pf_$pf.json 2> gpurun_out/l2pf_$pf.err; echo "pf=$pf rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])" gpurun_out/l2pf_$pf.json
done
NQ_JIT_L2PF=1 timeout 600 python -m pytest tests/test_sv_gpu.py tests/test_jit_gpu.py -x -q 2>&1 | tail -2
