set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
NQ_PLAN_TRACE=0 timeout 300 python scripts/dm_trace.py 14 2; echo "dm_trace rc=$?"
timeout 600 python scripts/secondary_probe.py > gpurun_out/secondary_probe.json 2> gpurun_out/secondary_probe.err; echo "probe rc=$?"
python -c "import json; d=json.load(open('gpurun_out/secondary_probe.json')); print({k:(v.get('device_ms'), v.get('passes')) for k,v in d.items() if k!='jit'})"
