run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/k3_$name.json 2> gpurun_out/k3_$name.err; echo "$name rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['secondary']; print(d['value'], d['roofline']['frac'], 'qft', s['qft30']['ms_per_circuit'], 'vqe', s['vqe28']['ms_per_eval'], 'dm14', s['dm_noisy_tfim14']['wall_s'], 'qaoa', s['dm_noisy_qaoa14']['wall_s'])" gpurun_out/k3_$name.json; }
run base NQ_X=0
run dskip NQ_DIAG_SKIP=1
run relabel0 NQ_RELABEL=0
