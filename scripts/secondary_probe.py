"""Break down the secondary workloads (VQE n=28, DM noisy TFIM n=14, QFT-30)
into planner stats and device-timed phases.  Run on the GPU box."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06861_b200 import abi, naqs, workloads  # noqa: E402


def timed(fn, reps=3):
    fn()
    abi.jit_wait()
    fn()
    abi.profile_begin(-1, per_pass_events=True)
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    wall = (time.perf_counter() - t0) / reps
    p = abi.profile_end(-1)
    return {"wall_ms": wall * 1e3, "device_ms": p["region_ms"] / reps, "pass_ms": p["pass_ms"] / reps,
            "passes": p["pass_launches"] / reps, "kernels": p["kernel_launches"] / reps}


out = {}
# VQE n = 28
nv, layers = 28, 3
vops = abi.make_ops(workloads.vqe_ansatz(nv, layers, workloads.vqe_initial_params(nv, layers)))
terms = workloads.tfim_hamiltonian(nv)
sv = abi.SV(nv)
out["vqe_apply"] = timed(lambda: (sv.reset(), sv.apply(vops).flush(), sv.synchronize()))
out["vqe_apply"]["stats"] = sv.stats()
out["vqe_expect55"] = timed(lambda: sv.expectations(terms))
out["vqe_reset"] = timed(lambda: (sv.reset(), sv.synchronize()))
sv.close()

# DM noisy TFIM n = 14
nd = 14
cal = {"name": "synthetic", "qubits": [{"t1_us": 60.0, "t2_us": 40.0, "readout_p01": 0.02, "readout_p10": 0.02}] * nd,
       "default_1q": {"error": 0.001, "duration_ns": 50.0}, "default_2q": {"error": 0.01, "duration_ns": 300.0}}
model = naqs.load_calibration(json.dumps(cal))
circ = naqs.Circuit(nd)
for name, qs, ps in workloads.tfim_trotter(nd, 1.0, steps=10):
    circ.add(name, qs, ps)
out["dm_tfim14"] = timed(lambda: naqs.density_expectation(circ, "Z" + "I" * (nd - 1), model), reps=2)

# QFT-30
qops = abi.make_ops(workloads.qft(30))
sv = abi.SV(30)
out["qft30"] = timed(lambda: (sv.apply(qops).flush(), sv.synchronize()), reps=2)
out["qft30"]["stats"] = sv.stats()
sv.close()
out["jit"] = abi.jit_stats()
print(json.dumps(out, indent=1))
