# round 2: full GPU suite after the DLPack fix, pivot-normalisation A/B, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d_pytest.log
for nd in 1 0 1; do NQ_NORM_DENSE=$nd timeout 300 python scripts/pass_timing.py >> gpurun_out/r2d_timing.jsonl 2>>gpurun_out/r2d_timing.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:nqjit --csv --log-file gpurun_out/r2d_launches_rand.csv python scripts/pass_timing.py rand > /dev/null 2>&1
tail -3 gpurun_out/r2d_pytest.log; cat gpurun_out/r2d_timing.jsonl
