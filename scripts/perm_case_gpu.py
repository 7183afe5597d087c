"""GPU side of the PX=0 bisect: run the permutation-heavy 12-qubit / tile-8
case of tests/test_jit_gpu.py, save the amplitudes (compare with
tests/jit_emu.py on the generated sources, NQ_JIT_DUMP)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
from oracle import Port  # noqa: E402
from paper_2401_06861_b200 import abi  # noqa: E402

port = Port()
prng = np.random.default_rng(99)
kinds = [("cx", 2, 0), ("cx", 2, 0), ("ccx", 3, 0), ("swap", 2, 0), ("x", 1, 0), ("y", 1, 0), ("ry", 1, 1),
         ("u3", 1, 3), ("h", 1, 0), ("t", 1, 0), ("rz", 1, 1), ("cz", 2, 0), ("s", 1, 0)]
n, tile = 12, 8
circ = []
for _ in range(300):
    k, ar, npar = kinds[int(prng.integers(len(kinds)))]
    qs = [int(q) for q in prng.choice(n, size=ar, replace=False)]
    circ.append((k, qs, [float(v) for v in prng.uniform(-3, 3, size=npar)]))
for layers in range(2):
    circ += [("cx", [i, i + 1], []) for i in range(n - 1)] + [("ry", [q], [0.1 * q + 0.3]) for q in range(n)]
sv = abi.SV(n, tile_qubits=tile)
sv.apply(abi.make_ops(circ))
got = sv.amplitudes()
tag = sys.argv[1] if len(sys.argv) > 1 else "x"
np.save(os.path.join(ROOT, "gpurun_out", f"perm12_{tag}.npy"), got)
print(tag, float(np.max(np.abs(got - port.sv_run(n, circ)))), sv.stats())
