for cfg in "4 11" "5 11" "6 11" "5 12" "6 12"; do
  set -- $cfg
  NQ_LOW_BITS=$1 timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-secondary --tile $2 > gpurun_out/lb2_$1_$2.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/lb2_$1_$2.json'));print('lowbits=$1 tile=$2', round(d['value']), 'gates/s', round(d['roofline']['avg_launch_ms'],2),'ms/pass', d['passes_per_step'],'passes')" || tail -3 gpurun_out/lb2_$1_$2.json
done
