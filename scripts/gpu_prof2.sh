set -x
timeout 600 python scripts/secondary_probe.py > gpurun_out/secondary_probe.json 2> gpurun_out/secondary_probe.err; echo "probe rc=$?"
cat gpurun_out/secondary_probe.json; tail -3 gpurun_out/secondary_probe.err
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/prof_plain.json 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nqjit -s 8 -c 2 -o gpurun_out/prof_jit_best python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_full.log
