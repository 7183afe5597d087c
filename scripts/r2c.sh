set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2c_pytest.log
timeout 300 python scripts/pass_timing.py > gpurun_out/r2c_timing.jsonl 2>gpurun_out/r2c_timing.err
timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
tail -3 gpurun_out/r2c_pytest.log; cat gpurun_out/r2c_timing.jsonl; tail -c 600 gpurun_out/r2c_bench.json
