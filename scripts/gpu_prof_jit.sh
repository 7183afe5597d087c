set -x
T=${TILE:-11}
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary --tile $T > gpurun_out/prof_plain.json 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nqjit -s 3 -c 2 -o gpurun_out/prof_jit_t$T python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary --tile $T > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_full.log
