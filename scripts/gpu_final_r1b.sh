set -x
start=$(date +%s); timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/final_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:nqjit -s 7 -c 7 -o gpurun_out/final_prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/final_ncu_full.log 2>&1; echo "ncu full rc=$?"
