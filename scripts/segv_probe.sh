for i in 1 2 3; do
NQ_SEGV_TRACE=1 timeout 300 python scripts/dm_trace.py 14 2 > gpurun_out/segv_t.txt 2>&1; echo "rc=$?"
done
tail -5 gpurun_out/segv_t.txt
