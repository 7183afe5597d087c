for cfg in "0 4 11" "0 5 11" "0 6 11" "0 6 10" "0 8 10" "1 4 10" "0 2 12" "0 3 12"; do
  set -- $cfg
  NQ_JIT_PREFETCH=$1 NQ_JIT_MINB=$2 timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-secondary --tile $3 > gpurun_out/sweep_$1_$2_$3.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/sweep_$1_$2_$3.json'));print('pf=$1 minb=$2 tile=$3', round(d['value']), 'gates/s', round(d['roofline']['avg_launch_ms'],2),'ms/pass', d['passes_per_step'],'passes')" || tail -3 gpurun_out/sweep_$1_$2_$3.json
done
