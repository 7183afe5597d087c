import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06861_b200 import abi, workloads
nv, layers = 28, 3
vops = abi.make_ops(workloads.vqe_ansatz(nv, layers, workloads.vqe_initial_params(nv, layers)))
sv = abi.SV(nv)
sv.apply(vops).flush(); abi.jit_wait()
for _ in range(2):
    sv.reset(); sv.apply(vops).flush(); sv.synchronize()
print("ok", abi.jit_stats())
