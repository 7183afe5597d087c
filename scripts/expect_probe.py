import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06861_b200 import abi, workloads
n = 30
sv = abi.SV(n)
sv.apply(abi.make_ops(workloads.random_circuit(2024, n, 200))).flush()
term = [("Z" + "I" * (n - 1), 1.0)]
for i in range(6):
    sv.synchronize()
    t = time.perf_counter()
    v = sv.expectations(term)
    dt = (time.perf_counter() - t) * 1e3
    print(f"expect call {i}: {dt:.2f} ms", v, abi.jit_stats(), flush=True)
    if i == 1:
        abi.jit_wait()
abi.profile_begin(-1, True)
for i in range(3):
    sv.expectations(term)
p = abi.profile_end(-1)
print("profiled", p["region_ms"] / 3, "ms/call, kernels", p["kernel_launches"] / 3)
