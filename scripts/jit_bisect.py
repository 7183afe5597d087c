"""Per-case errors of the specialised pass kernels vs the oracle (bisect helper).
    NQ_JIT=sync python scripts/jit_bisect.py      (env knobs apply)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
from oracle import Port  # noqa: E402
from paper_2401_06861_b200 import abi  # noqa: E402

port = Port()
env = {k: v for k, v in os.environ.items() if k.startswith("NQ_")}
for n, tile, seed in [(12, 8, 1), (14, 10, 2), (16, 12, 3), (18, 12, 4), (17, 9, 5), (20, 13, 6), (22, 11, 7)]:
    ops = port.random_circuit(seed, n, 250)
    sv = abi.SV(n, tile_qubits=tile)
    sv.apply(ops)
    err = float(np.max(np.abs(sv.amplitudes() - port.sv_run(n, ops))))
    print("random", n, tile, seed, f"{err:.3e}", env, flush=True)
prng = np.random.default_rng(99)
kinds = [("cx", 2, 0), ("cx", 2, 0), ("ccx", 3, 0), ("swap", 2, 0), ("x", 1, 0), ("y", 1, 0), ("ry", 1, 1),
         ("u3", 1, 3), ("h", 1, 0), ("t", 1, 0), ("rz", 1, 1), ("cz", 2, 0), ("s", 1, 0)]
for n, tile, seed in [(12, 8, 11), (15, 10, 12), (18, 11, 13), (21, 12, 14)]:
    circ = []
    for _ in range(300):
        k, ar, npar = kinds[int(prng.integers(len(kinds)))]
        qs = [int(q) for q in prng.choice(n, size=ar, replace=False)]
        circ.append((k, qs, [float(v) for v in prng.uniform(-3, 3, size=npar)]))
    for layers in range(2):
        circ += [("cx", [i, i + 1], []) for i in range(n - 1)] + [("ry", [q], [0.1 * q + 0.3]) for q in range(n)]
    sv = abi.SV(n, tile_qubits=tile)
    sv.apply(abi.make_ops(circ))
    err = float(np.max(np.abs(sv.amplitudes() - port.sv_run(n, circ))))
    print("perm", n, tile, seed, f"{err:.3e}", env, flush=True)
