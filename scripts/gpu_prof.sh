set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/prof_plain.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pass_kernel -s 3 -c 1 -o gpurun_out/prof_pass12 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -5 gpurun_out/ncu_full.log
