"""Device time per pass of the three SV benchmark workloads (A/B helper).

    python scripts/pass_timing.py [rand qft vqe]     (env knobs apply)
Prints one JSON line per workload: ms per circuit, passes, ms per pass,
fraction of the HBM roofline (32 * 2^n bytes per pass / MEASURED_PEAKS hbm_gbs).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_06861_b200 import abi, workloads  # noqa: E402

try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except OSError:
    PEAK = 6534.5


def run(name, n, ops, reps=3, extra=None):
    # every repetition starts from |0..0> in the identity layout (a flush
    # may end on a carried qubit layout, and a different layout is a
    # different plan); only the passes are timed
    arr = abi.make_ops(ops)
    sv = abi.SV(n)
    for _ in range(2):
        sv.reset()
        sv.apply(arr).flush()
        abi.jit_wait()
    sv.synchronize()
    pass_ms = 0.0
    launches = 0
    for _ in range(reps):
        sv.reset()
        sv.synchronize()
        abi.profile_begin(0, per_pass_events=True)
        sv.apply(arr).flush()
        if extra:
            extra(sv)
        p = abi.profile_end(0)
        pass_ms += p["pass_ms"]
        launches += p["pass_launches"]
    p = {"pass_ms": pass_ms, "pass_launches": launches, "region_ms": pass_ms}
    st = sv.stats()
    sv.close()
    per = p["pass_ms"] / max(p["pass_launches"], 1)
    out = {"workload": name, "ms_per_circuit": p["region_ms"] / reps, "passes": st["passes"], "ms_per_pass": per,
           "frac": (32 << n) / (per / 1e3) / 1e9 / PEAK, "env": {k: v for k, v in os.environ.items() if k.startswith("NQ_")}}
    print(json.dumps(out), flush=True)


sel = sys.argv[1:] or ["rand", "qft", "vqe"]
if "rand" in sel:
    run("random30", 30, workloads.random_circuit(2024, 30, 200))
if "qft" in sel:
    run("qft30", 30, workloads.qft(30))
if "vqe" in sel:
    nv = 28
    run("vqe28", nv, workloads.vqe_ansatz(nv, 3, workloads.vqe_initial_params(nv, 3)))
