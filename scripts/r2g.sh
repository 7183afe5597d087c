# full GPU suite + pass timing + launch list (normalisation, coalesced relabelled stores, 256-bit pairs, try_cancel fix)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2g_pytest.log
timeout 300 python scripts/pass_timing.py > gpurun_out/r2g_timing.jsonl 2>gpurun_out/r2g_timing.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:nqjit --csv --log-file gpurun_out/r2g_launches.csv python scripts/pass_timing.py > /dev/null 2>&1
tail -3 gpurun_out/r2g_pytest.log; cat gpurun_out/r2g_timing.jsonl
