for t in 11 12 10; do
NQ_TILE_SV=$t timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/tile_$t.json 2> gpurun_out/tile_$t.err; echo "tile=$t rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['secondary']; print(d['value'], d['ms_per_step'], d['passes_per_step'], d['roofline']['frac'], 'qft', s['qft30']['ms_per_circuit'], s['qft30']['passes_per_circuit'], 'vqe', s['vqe28']['ms_per_eval'], 'tr', s['trajectories']['tfim_n10_5steps']['gpu_wall_s'])" gpurun_out/tile_$t.json
done
for t in 12 10; do
NQ_TILE_DM=$t timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/tiledm_$t.json 2> gpurun_out/tiledm_$t.err; echo "tiledm=$t rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d['secondary']; print('dm14', s['dm_noisy_tfim14']['wall_s'], 'qaoa', s['dm_noisy_qaoa14']['wall_s'], 'dm16', s['dm_noisy_tfim16']['wall_s'])" gpurun_out/tiledm_$t.json
done
