timeout 300 python scripts/batch_probe.py 2>&1 | tail -12
timeout 300 python -c "
import time, sys
sys.path.insert(0,'.')
from paper_2401_06861_b200 import naqs, workloads, abi
cal=open('tests/golden/example_5q.json').read(); m=naqs.load_calibration(cal)
for i in range(5):
    t=time.perf_counter(); workloads.tfim_sweep_rows_batched(naqs,4,m); print('sweep', time.perf_counter()-t)
import cProfile, pstats
cProfile.run('workloads.tfim_sweep_rows_batched(naqs,4,m)', '/tmp/p.out')
pstats.Stats('/tmp/p.out').sort_stats('cumtime').print_stats(12)
" 2>&1 | tail -40
