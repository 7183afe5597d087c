mkdir -p gpurun_out
for cfg in "NQ_JIT_PX=0" "NQ_JIT_PX=0 NQ_NORM_DENSE=0" "NQ_JIT_PX=0 NQ_JIT_PHASEACC=0" "NQ_JIT_PX=1"; do
  env $cfg NQ_JIT=sync timeout 600 python scripts/jit_bisect.py >> gpurun_out/r2e_bisect.log 2>&1
done
cat gpurun_out/r2e_bisect.log
