"""Synthetic circuits of the BASELINE.json configurations.

Input generation only -- these build op lists, they compute nothing:
* random_circuit: the reference's seeded generator (proj/tests/test_util.hpp:59-86)
  restated over xoshiro256++ (proj/include/naqs/rng.hpp), so the same seed
  gives the same circuit as the reference's own tests;
* qft: QFT in the reference gate set (cp = u1, cx, u1, cx, u1), final swaps,
  after an RY/RZ layer drawn from Rng(7);
* tfim_trotter: build_trotter_circuit (proj/src/tfim.cpp:38-64);
* tfim_hamiltonian: build_tfim_hamiltonian (proj/src/tfim.cpp:12-36);
* qaoa_ring: QAOA-MaxCut ring, p layers;
* vqe_ansatz: build_ansatz_circuit (proj/src/vqe.cpp:14-30).
"""
from __future__ import annotations

import math
from typing import List, Tuple

M64 = (1 << 64) - 1


class Rng:
    """xoshiro256++ seeded through SplitMix64 (same stream as naqs::Rng)."""

    def __init__(self, seed: int):
        x = seed & M64
        self.s = []
        for _ in range(4):
            x = (x + 0x9E3779B97F4A7C15) & M64
            self.s.append(_mix(x))

    def next_u64(self) -> int:
        s = self.s
        r = (_rotl((s[0] + s[3]) & M64, 23) + s[0]) & M64
        t = (s[1] << 17) & M64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl(s[3], 45)
        return r

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()


def _rotl(x: int, k: int) -> int:
    return ((x << k) | (x >> (64 - k))) & M64


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


Op = Tuple[str, List[int], List[float]]
_POOL = ["x", "y", "z", "h", "s", "sdg", "t", "tdg", "id", "rx", "ry", "rz", "u1", "u2", "u3", "cx", "cz", "swap", "ccx"]
_ARITY = {"cx": 2, "cz": 2, "swap": 2, "ccx": 3}
_NPAR = {"rx": 1, "ry": 1, "rz": 1, "u1": 1, "u2": 2, "u3": 3}


def random_circuit(seed: int, n: int, depth: int, max_arity: int = 3) -> List[Op]:
    rng = Rng(seed)
    out: List[Op] = []
    for _ in range(depth):
        while True:
            kind = _POOL[rng.next_u64() % len(_POOL)]
            ar = _ARITY.get(kind, 1)
            if ar <= n and ar <= max_arity:
                break
        qs: List[int] = []
        while len(qs) < ar:
            q = rng.next_u64() % n
            if q not in qs:
                qs.append(int(q))
        params = [rng.uniform(-2.0 * math.pi, 2.0 * math.pi) for _ in range(_NPAR.get(kind, 0))]
        out.append((kind, qs, params))
    return out


def qft(n: int, prep_seed: int = 7) -> List[Op]:
    rng = Rng(prep_seed)
    ops: List[Op] = []
    for q in range(n):
        ops.append(("ry", [q], [rng.uniform(-math.pi, math.pi)]))
        ops.append(("rz", [q], [rng.uniform(-math.pi, math.pi)]))
    for j in reversed(range(n)):
        ops.append(("h", [j], []))
        for k in reversed(range(j)):
            lam = math.pi / (1 << (j - k))
            # controlled phase cp(lam) between control k and target j
            ops.append(("u1", [k], [lam / 2]))
            ops.append(("cx", [k, j], []))
            ops.append(("u1", [j], [-lam / 2]))
            ops.append(("cx", [k, j], []))
            ops.append(("u1", [j], [lam / 2]))
    for q in range(n // 2):
        ops.append(("swap", [q, n - 1 - q], []))
    return ops


def tfim_trotter(n: int, t: float, steps_per_unit: int = 100, J: float = 1.0, h: float = 1.0,
                 periodic: bool = False, steps: int | None = None) -> List[Op]:
    if t == 0.0:
        return []
    nsteps = steps if steps is not None else int(math.ceil(t * steps_per_unit))
    delta = t / nsteps
    bonds = [(i, i + 1) for i in range(n - 1)]
    if periodic and n >= 3:
        bonds.append((n - 1, 0))
    ops: List[Op] = []
    for _ in range(nsteps):
        for i, j in bonds:
            ops += [("cx", [i, j], []), ("rz", [j], [-2.0 * J * delta]), ("cx", [i, j], [])]
        for i in range(n):
            ops.append(("rx", [i], [-2.0 * h * delta]))
    return ops


def tfim_hamiltonian(n: int, J: float = 1.0, h: float = 1.0, periodic: bool = False):
    terms = []
    for i in range(n - 1):
        L = ["I"] * n
        L[i] = L[i + 1] = "Z"
        terms.append(("".join(L), -J))
    if periodic and n >= 3:
        L = ["I"] * n
        L[n - 1] = L[0] = "Z"
        terms.append(("".join(L), -J))
    for i in range(n):
        L = ["I"] * n
        L[i] = "X"
        terms.append(("".join(L), -h))
    return terms


def qaoa_ring(n: int, p: int = 2, gamma: float = 0.4, beta: float = 0.7) -> List[Op]:
    ops: List[Op] = [("h", [q], []) for q in range(n)]
    for _ in range(p):
        for i in range(n):
            j = (i + 1) % n
            ops += [("cx", [i, j], []), ("rz", [j], [2 * gamma]), ("cx", [i, j], [])]
        for q in range(n):
            ops.append(("rx", [q], [2 * beta]))
    return ops


def vqe_ansatz(n: int, layers: int, params) -> List[Op]:
    params = list(params)
    assert len(params) == n * (layers + 1)
    k = 0
    ops: List[Op] = []
    for q in range(n):
        ops.append(("ry", [q], [params[k]]))
        k += 1
    for _ in range(layers):
        for i in range(n - 1):
            ops.append(("cx", [i, i + 1], []))
        for q in range(n):
            ops.append(("ry", [q], [params[k]]))
            k += 1
    return ops


def vqe_initial_params(n: int, layers: int, seed: int = 1):
    """proj/src/vqe.cpp:123-125: Rng(seed).uniform(-0.1, 0.1) per parameter."""
    rng = Rng(seed)
    return [rng.uniform(-0.1, 0.1) for _ in range(n * (layers + 1))]


def tfim_sweep_times(t_max: float = 3.0, dt: float = 0.1):
    """Row times of magnetization_sweep (proj/src/tfim.cpp:158): t += dt from 0
    while t <= t_max + 1e-12 (accumulated, so 3.0 appears as 3.0000000000000013)."""
    out = []
    t = 0.0
    while t <= t_max + 1e-12:
        out.append(t)
        t += dt
    return out


def tfim_sweep_rows(naqs, n: int, model, t_max: float = 3.0, dt: float = 0.1, steps_per_unit: int = 100):
    """C1 driver over the drop-in API: (t, ideal <Z>, noisy <Z> after readout)
    per row of magnetization_sweep (proj/src/tfim.cpp:139-184, shots = 0,
    without the dense exact column)."""
    zs = []
    for q in range(n):
        L = ["I"] * n
        L[q] = "Z"
        zs.append("".join(L))
    rows = []
    for t in tfim_sweep_times(t_max, dt):
        c = naqs.Circuit(n)
        for name, qs, ps in tfim_trotter(n, t, steps_per_unit):
            c.add(name, qs, ps)
        ideal = sum(naqs.expectations(c, zs)) / n
        dist = naqs.noisy_distribution(c, model)
        noisy = 0.0
        for q in range(n):
            noisy += sum(-p if (i >> q) & 1 else p for i, p in enumerate(dist))
        rows.append((t, ideal, noisy / n))
    return rows


def tfim_sweep_rows_batched(naqs, n: int, model, t_max: float = 3.0, dt: float = 0.1, steps_per_unit: int = 100):
    """tfim_sweep_rows with every row's ideal circuit in one launch and every
    row's noisy density matrix in another (naqs.batch_* )."""
    import numpy as np

    zs = []
    for q in range(n):
        L = ["I"] * n
        L[q] = "Z"
        zs.append("".join(L))
    times = tfim_sweep_times(t_max, dt)
    circs = []
    for t in times:
        c = naqs.Circuit(n)
        for name, qs, ps in tfim_trotter(n, t, steps_per_unit):
            c.add(name, qs, ps)
        circs.append(c)
    ideal = naqs.batch_expectations(circs, zs).sum(axis=1) / n
    dists = naqs.batch_noisy_distributions(circs, model)
    sign = np.array([[-1.0 if (i >> q) & 1 else 1.0 for i in range(1 << n)] for q in range(n)])
    noisy = (dists @ sign.T).sum(axis=1) / n
    return [(t, float(a), float(b)) for t, a, b in zip(times, ideal, noisy)]
