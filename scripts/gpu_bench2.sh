set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for t in 12 11; do
timeout 600 python bench.py --no-cpu-baseline --tile $t > gpurun_out/bench_t$t.json 2> gpurun_out/bench_t$t.err; echo "bench $t rc=$?"
cat gpurun_out/bench_t$t.json; tail -3 gpurun_out/bench_t$t.err
done
