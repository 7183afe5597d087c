NQ_JIT_TMA=1 timeout 900 python -m pytest tests/test_jit_gpu.py tests/test_sv_gpu.py -x -q 2>&1 | tail -2
for t in 1 0; do
  NQ_JIT_TMA=$t timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/tma_$t.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/tma_$t.json'));s=d['secondary'];print('tma=$t', round(d['value']), 'gates/s', round(d['roofline']['avg_launch_ms'],2),'ms/pass; qft', round(s['qft30']['ms_per_circuit'],1), 'vqe', round(s['vqe28']['ms_per_eval'],2), 'dm', round(s['dm_noisy_tfim14']['wall_s']*1e3,1))" || tail -5 gpurun_out/tma_$t.json
done
NQ_JIT_TMA=1 python scripts/pattern_probe.py | tail -5
