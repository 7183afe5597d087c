nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/c1_clocks.csv &
SMI=$!
NQ_BATCH_TIMING=1 timeout 300 python scripts/batch_probe.py > gpurun_out/c1_probe.log 2>&1
kill $SMI
tail -30 gpurun_out/c1_probe.log
awk -F, '{print $2, $3, $4, $5}' gpurun_out/c1_clocks.csv | sort | uniq -c | sort -rn | head -20
