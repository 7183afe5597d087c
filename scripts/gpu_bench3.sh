set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for c in 1 0; do
NQ_COALESCE=$c timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-secondary > gpurun_out/coal_$c.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/coal_$c.json'));print('coalesce=$c', round(d['value']), 'gates/s', round(d['roofline']['avg_launch_ms'],2),'ms/pass', d['passes_per_step'],'passes', d['e2e']['value'])" || tail -3 gpurun_out/coal_$c.json
done
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
cat gpurun_out/bench_full.json
