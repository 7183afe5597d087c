"""Noisy TFIM density matrix (bench.py's dm_noisy_tfim14 workload) run three
times with its kernels compiled: the target of the DM ncu capture
(profiles/) -- the third call's passes are the Hermitian mirror passes.

    python scripts/dm_passes.py [n]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_06861_b200 import abi, workloads  # noqa: E402
from paper_2401_06861_b200 import naqs  # noqa: E402

nd = int(sys.argv[1]) if len(sys.argv) > 1 else 14
cal = {"name": "synthetic", "qubits": [{"t1_us": 60.0, "t2_us": 40.0, "readout_p01": 0.02, "readout_p10": 0.02}] * nd,
       "default_1q": {"error": 0.001, "duration_ns": 50.0}, "default_2q": {"error": 0.01, "duration_ns": 300.0}}
model = naqs.load_calibration(json.dumps(cal))
c = naqs.Circuit(nd)
for name, qs, ps in workloads.tfim_trotter(nd, 1.0, steps=10):
    c.add(name, qs, ps)
z = "Z" + "I" * (nd - 1)
naqs.density_expectation(c, z, model, max_qubits=nd)
abi.jit_wait()
naqs.density_expectation(c, z, model, max_qubits=nd)
abi.profile_begin(0, per_pass_events=True)
v = naqs.density_expectation(c, z, model, max_qubits=nd)
p = abi.profile_end(0)
print(json.dumps({"n": nd, "z0": v, "pass_launches": p["pass_launches"], "pass_ms": p["pass_ms"],
                  "bytes_per_launch": p["pass_bytes"] / max(p["pass_launches"], 1), "jit": abi.jit_stats()}))
