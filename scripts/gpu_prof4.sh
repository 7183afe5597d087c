timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/p4_plain.json 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nqjit -s 7 -c 7 -o gpurun_out/prof_relabel python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/p4_ncu.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/p4_ncu.log
