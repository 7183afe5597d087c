import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2401_06861_b200 import abi, naqs, workloads
n = 4
times = workloads.tfim_sweep_times()
circs = [[("gate", g) for g in workloads.tfim_trotter(n, t)] for t in times]
zs = [("Z" + "I" * (n - 1), 1.0)]
abi.batch_run(n, circs, zs)
for rep in range(3):
    t0 = time.perf_counter()
    abi.profile_begin(-1, False)
    abi.batch_run(n, circs, zs)
    p = abi.profile_end(-1)
    print("sv batch_run total", (time.perf_counter() - t0) * 1e3, "ms; device region", p["region_ms"], "ms")
arr, pool = abi.make_schedule([it for c in circs for it in c])
t0 = time.perf_counter(); abi.make_schedule([it for c in circs for it in c]); print("make_schedule ms", (time.perf_counter()-t0)*1e3)
cal = open("tests/golden/example_5q.json").read(); m = naqs.load_calibration(cal)
cc = []
for t in times:
    c = naqs.Circuit(n)
    for g, q, ps in workloads.tfim_trotter(n, t):
        c.add(g, q, ps)
    cc.append(c)
for rep in range(3):
    t0 = time.perf_counter()
    abi.profile_begin(-1, False)
    naqs.batch_noisy_distributions(cc, m)
    p = abi.profile_end(-1)
    print("dm batch total", (time.perf_counter() - t0) * 1e3, "ms; device region", p["region_ms"], "ms")
for rep in range(2):
    t0 = time.perf_counter()
    naqs.batch_expectations(cc, ["Z" + "I" * (n - 1)])
    print("sv naqs batch", (time.perf_counter() - t0) * 1e3, "ms")
