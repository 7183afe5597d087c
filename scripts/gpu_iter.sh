# Iteration check: GPU parity tests, headline bench (no CPU leg), secondary probe.
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/iter_bench.json 2> gpurun_out/iter_bench.err; echo "bench rc=$?"
cat gpurun_out/iter_bench.json; tail -3 gpurun_out/iter_bench.err
timeout 600 python scripts/secondary_probe.py > gpurun_out/secondary_probe.json 2> gpurun_out/secondary_probe.err; echo "probe rc=$?"
cat gpurun_out/secondary_probe.json; tail -3 gpurun_out/secondary_probe.err
