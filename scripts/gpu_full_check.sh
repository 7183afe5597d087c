set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/fc_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fc_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/fc_pytest.log
start=$(date +%s); timeout 900 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
cat gpurun_out/fc_bench.json
