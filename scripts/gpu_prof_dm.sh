timeout 300 python scripts/dm_trace.py 14 10 > gpurun_out/p5_dm.log 2>&1; echo "dm rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nqjit -s 10 -c 3 -o gpurun_out/prof_dm_pass python scripts/dm_trace.py 14 10 > gpurun_out/p5_ncu_dm.log 2>&1; echo "ncu dm rc=$?"
tail -2 gpurun_out/p5_ncu_dm.log
