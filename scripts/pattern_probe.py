"""Pass time vs tile bit placement (memory access pattern of the pass kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06861_b200 import abi
n = 30
sv = abi.SV(n)
for label, qs in [("high 4..10", range(4, 11)), ("high 12..18", range(12, 19)), ("high 23..29", range(23, 30)),
                  ("scattered", [5, 9, 13, 17, 21, 25, 29]), ("low-only 0..3", range(0, 4))]:
    ops = abi.make_ops([("h", [q], []) for q in qs] + [("h", [q], []) for q in qs])
    sv.apply(ops).flush(); abi.jit_wait(); sv.apply(ops).flush(); sv.synchronize()
    abi.profile_begin(-1, True)
    for _ in range(5):
        sv.apply(ops).flush()
    p = abi.profile_end(-1)
    ms = p["pass_ms"] / p["pass_launches"]
    print(f"{label:16s} passes/flush {p['pass_launches']/5:.0f}  {ms:.2f} ms/pass  {34.36/ms:.0f} GB/s  jit {abi.jit_stats()['launches']}")
