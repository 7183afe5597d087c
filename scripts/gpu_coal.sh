for c in 0 1; do
  NQ_COALESCE=$c timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-secondary > gpurun_out/coal_$c.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/coal_$c.json'));print('coalesce=$c', round(d['value']), 'gates/s', round(d['roofline']['avg_launch_ms'],2),'ms/pass', d['passes_per_step'],'passes')" || tail -3 gpurun_out/coal_$c.json
done
NQ_COALESCE=1 python scripts/pattern_probe.py | tail -1
