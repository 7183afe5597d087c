mkdir -p gpurun_out/dump_px0 gpurun_out/dump_px1
NQ_JIT=sync NQ_JIT_PX=0 NQ_JIT_DUMP=gpurun_out/dump_px0 python scripts/perm_case_gpu.py px0 > gpurun_out/r2f.log 2>&1
NQ_JIT=sync NQ_JIT_PX=1 NQ_JIT_DUMP=gpurun_out/dump_px1 python scripts/perm_case_gpu.py px1 >> gpurun_out/r2f.log 2>&1
NQ_JIT=off python scripts/perm_case_gpu.py off >> gpurun_out/r2f.log 2>&1
NQ_JIT=sync NQ_JIT_PX=0 NQ_NORM_DENSE=0 python scripts/perm_case_gpu.py px0nn >> gpurun_out/r2f.log 2>&1
NQ_JIT=sync NQ_JIT_PX=0 compute-sanitizer --tool racecheck python scripts/perm_case_gpu.py px0rc > gpurun_out/r2f_race.log 2>&1
cat gpurun_out/r2f.log; tail -5 gpurun_out/r2f_race.log
