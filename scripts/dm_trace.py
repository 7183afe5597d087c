"""Plan trace of the DM noisy TFIM-14 workload (run with NQ_PLAN_TRACE=1)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06861_b200 import abi, naqs, workloads  # noqa: E402

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 14
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cal = {"name": "synthetic", "qubits": [{"t1_us": 60.0, "t2_us": 40.0, "readout_p01": 0.02, "readout_p10": 0.02}] * nd,
       "default_1q": {"error": 0.001, "duration_ns": 50.0}, "default_2q": {"error": 0.01, "duration_ns": 300.0}}
model = naqs.load_calibration(json.dumps(cal))
circ = naqs.Circuit(nd)
for name, qs, ps in workloads.tfim_trotter(nd, 1.0, steps=steps):
    circ.add(name, qs, ps)
print(naqs.density_expectation(circ, "Z" + "I" * (nd - 1), model))
abi.jit_wait()  # second run uses the specialised pass kernels
print(naqs.density_expectation(circ, "Z" + "I" * (nd - 1), model))
print("jit", abi.jit_stats())
