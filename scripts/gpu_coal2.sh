for cfg in "0 0x1F" "1 0x1" "1 0x3" "1 0xF"; do
  set -- $cfg
  NQ_COALESCE=$1 NQ_COALESCE_MASK=$2 timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/coal_$1_$2.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/coal_$1_$2.json'));s=d['secondary'];print('coalesce=$1 mask=$2', round(d['value']), 'gates/s', round(d['roofline']['avg_launch_ms'],2),'ms/pass', d['passes_per_step'],'passes; qft', round(s['qft30']['ms_per_circuit'],1), 'vqe', round(s['vqe28']['ms_per_eval'],2), 'dm', round(s['dm_noisy_tfim14']['wall_s']*1e3,1))" || tail -3 gpurun_out/coal_$1_$2.json
done
