set -x
timeout 900 python -m pytest tests/test_jit_gpu.py tests/test_sv_gpu.py tests/test_scale_parity_gpu.py tests/test_dlpack_gpu.py -x -q -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
for acc in 1 0; do NQ_JIT_PHASEACC=$acc timeout 300 python scripts/pass_timing.py >> gpurun_out/r2b_timing.jsonl 2>>gpurun_out/r2b_timing.err; done
tail -3 gpurun_out/r2b_pytest.log; cat gpurun_out/r2b_timing.jsonl
