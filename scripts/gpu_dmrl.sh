timeout 900 python -m pytest tests/test_dm_gpu.py tests/test_jit_gpu.py tests/test_golden_gpu.py tests/test_batch_gpu.py -x -q 2>&1 | tail -2
for rl in 1 0; do
NQ_DM_RELABEL=$rl timeout 300 python - <<PY
import json, sys, time; sys.path.insert(0, '.')
from paper_2401_06861_b200 import abi, naqs, workloads
nd = 14
cal = {"name": "synthetic", "qubits": [{"t1_us": 60.0, "t2_us": 40.0, "readout_p01": 0.02, "readout_p10": 0.02}] * nd,
       "default_1q": {"error": 0.001, "duration_ns": 50.0}, "default_2q": {"error": 0.01, "duration_ns": 300.0}}
model = naqs.load_calibration(json.dumps(cal))
circ = naqs.Circuit(nd)
for name, qs, ps in workloads.tfim_trotter(nd, 1.0, steps=10):
    circ.add(name, qs, ps)
v = naqs.density_expectation(circ, "Z" + "I" * (nd - 1), model); abi.jit_wait()
naqs.density_expectation(circ, "Z" + "I" * (nd - 1), model)
abi.profile_begin(-1, True)
for _ in range(3): naqs.density_expectation(circ, "Z" + "I" * (nd - 1), model)
p = abi.profile_end(-1)
print("dmrelabel=$rl dm", round(p["region_ms"]/3, 1), "ms", p["pass_launches"]/3, "passes", round(p["pass_ms"]/p["pass_launches"], 3), "ms/pass", v, abi.jit_stats())
PY
done
