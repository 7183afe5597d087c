set -x
start=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
cat gpurun_out/bench_default.json; 
start=$(date +%s); timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - start ))s"
cat gpurun_out/bench_ref.json; 
