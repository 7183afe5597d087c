set -x
timeout 900 python -m pytest tests/test_jit_gpu.py tests/test_sv_gpu.py tests/test_scale_parity_gpu.py tests/test_dlpack_gpu.py -x -q -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
for acc in 1 0; do NQ_JIT_PHASEACC=$acc timeout 300 python scripts/pass_timing.py >> gpurun_out/r2b_timing.jsonl 2>>gpurun_out/r2b_timing.err; done
tail -3 gpurun_out/r2b_pytest.log; cat gpurun_out/r2b_timing.jsonl
ncu --set full --import-source on --clock-control none -k regex:nqjit --launch-skip 10 --launch-count 10 -o gpurun_out/r2b_qft -f python scripts/pass_timing.py qft > gpurun_out/r2b_ncu_qft.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:nqjit --launch-skip 7 --launch-count 7 -o gpurun_out/r2b_rand -f python scripts/pass_timing.py rand > gpurun_out/r2b_ncu_rand.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:nqjit --launch-skip 6 --launch-count 6 -o gpurun_out/r2b_vqe -f python scripts/pass_timing.py vqe > gpurun_out/r2b_ncu_vqe.log 2>&1
ls -la gpurun_out/
