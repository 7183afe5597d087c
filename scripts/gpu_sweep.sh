for cfg in "4 11 -1" "4 12 -1" "4 12 2" "4 11 3" "4 11 5"; do
  set -- $cfg
  NQ_REGBITS=$1 NQ_JIT_MINB=$3 timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-secondary --tile $2 > gpurun_out/sw_$1_$2_$3.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/sw_$1_$2_$3.json'));print('regbits=$1 tile=$2 minb=$3', round(d['value']), 'gates/s', round(d['roofline']['avg_launch_ms'],2),'ms/pass', d['passes_per_step'],'passes', 'jit', d['jit'])" || tail -3 gpurun_out/sw_$1_$2_$3.json
done
