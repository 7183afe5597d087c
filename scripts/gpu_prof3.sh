set -x
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/p3_plain.json 2>&1; echo "plain rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/p3_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 600 python scripts/secondary_probe.py > gpurun_out/p3_probe.json 2>&1; echo "probe rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:nqexp -s 3 -c 1 -o gpurun_out/prof_nqexp python scripts/secondary_probe.py > gpurun_out/p3_ncu_exp.log 2>&1; echo "ncu exp rc=$?"
timeout 300 python scripts/dm_trace.py 14 10 > gpurun_out/p3_dm.log 2>&1; echo "dm rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:nqjit -s 60 -c 1 -o gpurun_out/prof_dm_pass python scripts/dm_trace.py 14 10 > gpurun_out/p3_ncu_dm.log 2>&1; echo "ncu dm rc=$?"
tail -3 gpurun_out/p3_ncu_exp.log gpurun_out/p3_ncu_dm.log
