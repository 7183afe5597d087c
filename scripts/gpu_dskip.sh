for v in 0 1; do
  NQ_DIAG_SKIP=$v timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/dskip_$v.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/dskip_$v.json'));s=d['secondary'];print('diagskip=$v', round(d['value']), 'gates/s', round(d['roofline']['avg_launch_ms'],2),'ms/pass; qft', round(s['qft30']['ms_per_circuit'],1), 'vqe', round(s['vqe28']['ms_per_eval'],2), 'dm', round(s['dm_noisy_tfim14']['wall_s']*1e3,1))" || tail -3 gpurun_out/dskip_$v.json
done
