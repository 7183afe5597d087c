run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/k2_$name.json 2> gpurun_out/k2_$name.err; echo "$name rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['secondary']; print(d['value'], d['ms_per_step'], d['passes_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], 'qft', s['qft30']['ms_per_circuit'], 'vqe', s['vqe28']['ms_per_eval'], 'dm14', s['dm_noisy_tfim14']['wall_s'])" gpurun_out/k2_$name.json; }
run base NQ_X=0
run rb3 NQ_REGBITS=3
run rb3_t12 NQ_REGBITS=3 NQ_TILE_SV=12
run rb3_t10 NQ_REGBITS=3 NQ_TILE_SV=10
