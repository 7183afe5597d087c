for lb in 4 3 2 1 0; do
  NQ_LOW_BITS=$lb timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-secondary > gpurun_out/lb_$lb.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/lb_$lb.json'));print('lowbits=$lb', round(d['value']), 'gates/s', round(d['roofline']['avg_launch_ms'],2),'ms/pass', d['passes_per_step'],'passes')" || tail -3 gpurun_out/lb_$lb.json
done
for lb in 4 2 1; do
NQ_LOW_BITS=$lb timeout 300 python - <<PY
import sys, time; sys.path.insert(0, '.')
from paper_2401_06861_b200 import abi, workloads
sv = abi.SV(30); ops = abi.make_ops(workloads.qft(30))
sv.apply(ops).flush(); abi.jit_wait(); sv.apply(ops).flush(); sv.synchronize()
abi.profile_begin(-1, True)
for _ in range(2): sv.apply(ops).flush()
p = abi.profile_end(-1)
print("qft lowbits=$lb", round(p["region_ms"]/2, 1), "ms", p["pass_launches"]/2, "passes", round(p["pass_ms"]/p["pass_launches"], 2), "ms/pass")
PY
done
