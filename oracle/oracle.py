"""TEST INFRASTRUCTURE ONLY -- Python handles on the two CPU checkers.

* ``Port``  -- oracle/_build/liboracle.so, the C restatement (naqs_oracle.c).
* ``Ref``   -- oracle/_ref/libnaqs_ref.so, the reference's own sources
  compiled unmodified (oracle/Makefile); present when it was built in the
  container that has /root/reference (the .so travels with the repo).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(_HERE, "_build", "liboracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libnaqs_ref.so")

KINDS = [
    "x", "y", "z", "h", "s", "sdg", "t", "tdg", "id",
    "rx", "ry", "rz", "u1", "u2", "u3",
    "cx", "cz", "swap", "ccx", "measure", "barrier",
]
OP_DTYPE = np.dtype(
    [("kind", "<i4"), ("nqubits", "<i4"), ("qubits", "<i4", (3,)), ("reserved", "<i4"), ("params", "<f8", (3,))],
    align=True,
)

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


def _d(a):
    return a.ctypes.data_as(_dp)


def _c(a):
    return a.view(np.float64).ctypes.data_as(_dp)


def ops_to_list(arr: np.ndarray):
    out = []
    for o in arr:
        name = KINDS[int(o["kind"])]
        k = int(o["nqubits"])
        npar = {"rx": 1, "ry": 1, "rz": 1, "u1": 1, "u2": 2, "u3": 3}.get(name, 0)
        out.append((name, [int(q) for q in o["qubits"][:k]], [float(p) for p in o["params"][:npar]]))
    return out


def list_to_ops(ops) -> np.ndarray:
    arr = np.zeros(len(ops), dtype=OP_DTYPE)
    for i, op in enumerate(ops):
        arr[i]["kind"] = KINDS.index(op[0])
        arr[i]["nqubits"] = len(op[1])
        for j, q in enumerate(op[1]):
            arr[i]["qubits"][j] = q
        for j, p in enumerate(op[2] if len(op) > 2 else ()):
            arr[i]["params"][j] = p
    return arr


class _Noise(C.Structure):
    _fields_ = [("t1", _dp), ("t2", _dp), ("p01", _dp), ("p10", _dp),
                ("e1", C.c_double), ("d1", C.c_double), ("e2", C.c_double), ("d2", C.c_double)]


class NoiseSpec:
    """Synthetic uniform calibration: per-qubit T1/T2/readout
    and default_1q / default_2q gate entries."""

    def __init__(self, n, t1=60.0, t2=40.0, p01=0.02, p10=0.02, e1=0.001, d1=50.0, e2=0.01, d2=300.0):
        self.n = n
        self.t1 = np.full(n, t1, dtype=np.float64)
        self.t2 = np.full(n, t2, dtype=np.float64)
        self.p01 = np.full(n, p01, dtype=np.float64)
        self.p10 = np.full(n, p10, dtype=np.float64)
        self.e1, self.d1, self.e2, self.d2 = e1, d1, e2, d2

    def arrays(self):
        return _d(self.t1), _d(self.t2), _d(self.p01), _d(self.p10)

    def calibration_json(self) -> str:
        import json
        return json.dumps({
            "name": "synthetic",
            "qubits": [{"t1_us": float(self.t1[q]), "t2_us": float(self.t2[q]),
                        "readout_p01": float(self.p01[q]), "readout_p10": float(self.p10[q])} for q in range(self.n)],
            "default_1q": {"error": self.e1, "duration_ns": self.d1},
            "default_2q": {"error": self.e2, "duration_ns": self.d2},
        })


class Port:
    """The C restatement (oracle/naqs_oracle.c)."""

    def __init__(self, path: str = PORT_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run __graft_entry__.build()")
        self.lib = C.CDLL(path)
        L = self.lib
        L.or_derive_seed.restype = C.c_uint64
        L.or_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        for f in ("or_sv_norm_sq", "or_sv_expectation", "or_dm_trace", "or_dm_purity", "or_dm_hermiticity"):
            getattr(L, f).restype = C.c_double
        L.or_sv_expectation.argtypes = [_dp, C.c_int, C.c_char_p, C.c_double]
        L.or_rng_u64.argtypes = [C.c_uint64, C.c_int, _u64p]
        L.or_rng_double.argtypes = [C.c_uint64, C.c_int, _dp]
        L.or_random_circuit.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.or_sample_distribution.argtypes = [_dp, C.c_int, C.c_uint64, C.c_uint64, _u64p]
        L.or_dm_expectation.argtypes = [_dp, C.c_int, C.c_char_p, C.c_double, _dp]
        L.or_readout_apply_dist.argtypes = [_dp, C.c_int, _dp, _dp, _dp]
        L.or_dm_run_noisy.argtypes = [_dp, C.c_int, C.c_void_p, C.c_int64, C.POINTER(_Noise)]
        L.or_sv_apply.argtypes = [_dp, C.c_int, C.c_void_p, C.c_int64]
        L.or_dm_apply.argtypes = [_dp, C.c_int, C.c_void_p, C.c_int64]
        L.or_depolarizing.argtypes = [C.c_double, C.c_int, _dp]
        L.or_thermal_relaxation.argtypes = [C.c_double, C.c_double, C.c_double, _dp]
        L.or_amplitude_damping.argtypes = [C.c_double, _dp]
        L.or_dm_apply_operators.argtypes = [_dp, C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, _dp]
        L.or_sv_apply_matrix.argtypes = [_dp, C.c_int, C.POINTER(C.c_int), C.c_int, _dp]
        L.or_sv_kraus_trajectory.argtypes = [_dp, C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, _dp, _u64p]
        L.or_rng_init.argtypes = [_u64p, C.c_uint64]
        L.or_gate_matrix.argtypes = [C.c_void_p, _dp]

    # --- rng / generators
    def rng_u64(self, seed, count):
        out = np.zeros(count, dtype=np.uint64)
        self.lib.or_rng_u64(seed, count, out.ctypes.data_as(_u64p))
        return out

    def rng_double(self, seed, count):
        out = np.zeros(count)
        self.lib.or_rng_double(seed, count, _d(out))
        return out

    def derive_seed(self, base, stream):
        return int(self.lib.or_derive_seed(base, stream))

    def random_circuit(self, seed, n, depth, max_arity=3) -> np.ndarray:
        out = np.zeros(depth, dtype=OP_DTYPE)
        self.lib.or_random_circuit(seed, n, depth, max_arity, out.ctypes.data)
        return out

    def gate_matrix(self, op) -> np.ndarray:
        arr = list_to_ops([op])
        m = np.zeros(64, dtype=np.complex128)
        d = self.lib.or_gate_matrix(arr.ctypes.data, _c(m))
        return m[: d * d].reshape(d, d)

    # --- state vector
    def sv_run(self, n, ops) -> np.ndarray:
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        a = np.zeros(1 << n, dtype=np.complex128)
        a[0] = 1.0
        if self.lib.or_sv_apply(_c(a), n, arr.ctypes.data, len(arr)) != 0:
            raise ValueError("MEASURE in state-vector run")
        return a

    def sv_apply(self, amps, ops):
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        n = int(np.log2(len(amps)))
        self.lib.or_sv_apply(_c(amps), n, arr.ctypes.data, len(arr))
        return amps

    def sv_apply_matrix(self, amps, qubits, mat):
        q = (C.c_int * len(qubits))(*qubits)
        m = np.ascontiguousarray(mat, dtype=np.complex128)
        self.lib.or_sv_apply_matrix(_c(amps), int(np.log2(len(amps))), q, len(qubits), _c(m))

    def norm_sq(self, amps):
        return self.lib.or_sv_norm_sq(_c(amps), int(np.log2(len(amps))))

    def expectation(self, amps, letters, coeff=1.0):
        return self.lib.or_sv_expectation(_c(amps), int(np.log2(len(amps))), letters.encode(), coeff)

    def sample_distribution(self, dist, shots, seed):
        d = np.ascontiguousarray(dist, dtype=np.float64)
        n = int(np.log2(len(d)))
        out = np.zeros(len(d), dtype=np.uint64)
        self.lib.or_sample_distribution(_d(d), n, shots, seed, out.ctypes.data_as(_u64p))
        return out

    def kraus_trajectory(self, amps, qubits, kraus, rng_state):
        q = (C.c_int * len(qubits))(*qubits)
        k = np.ascontiguousarray(kraus, dtype=np.complex128)
        return self.lib.or_sv_kraus_trajectory(_c(amps), int(np.log2(len(amps))), q, len(qubits), len(k), _c(k),
                                               rng_state.ctypes.data_as(_u64p))

    def rng_state(self, seed):
        s = np.zeros(4, dtype=np.uint64)
        self.lib.or_rng_init(s.ctypes.data_as(_u64p), seed)
        return s

    # --- density matrix
    def dm_new(self, n):
        rho = np.zeros(1 << (2 * n), dtype=np.complex128)
        rho[0] = 1.0
        return rho

    def dm_run(self, n, ops) -> np.ndarray:
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        rho = self.dm_new(n)
        self.lib.or_dm_apply(_c(rho), n, arr.ctypes.data, len(arr))
        return rho.reshape(1 << n, 1 << n)

    def dm_apply_channel(self, rho, qubits, kraus):
        n = int(np.log2(rho.shape[0]))
        flat = np.ascontiguousarray(rho.reshape(-1))
        q = (C.c_int * len(qubits))(*qubits)
        k = np.ascontiguousarray(kraus, dtype=np.complex128)
        self.lib.or_dm_apply_operators(_c(flat), n, q, len(qubits), len(k), _c(k))
        return flat.reshape(rho.shape)

    def dm_run_noisy(self, n, ops, noise: NoiseSpec) -> np.ndarray:
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        rho = self.dm_new(n)
        t1, t2, p01, p10 = noise.arrays()
        spec = _Noise(t1, t2, p01, p10, noise.e1, noise.d1, noise.e2, noise.d2)
        if self.lib.or_dm_run_noisy(_c(rho), n, arr.ctypes.data, len(arr), C.byref(spec)) != 0:
            raise ValueError("gate not calibratable")
        return rho.reshape(1 << n, 1 << n)

    def dm_trace(self, rho):
        return self.lib.or_dm_trace(_c(np.ascontiguousarray(rho.reshape(-1))), int(np.log2(rho.shape[0])))

    def dm_purity(self, rho):
        return self.lib.or_dm_purity(_c(np.ascontiguousarray(rho.reshape(-1))), int(np.log2(rho.shape[0])))

    def dm_hermiticity(self, rho):
        return self.lib.or_dm_hermiticity(_c(np.ascontiguousarray(rho.reshape(-1))), int(np.log2(rho.shape[0])))

    def dm_expectation(self, rho, letters, coeff=1.0):
        out = C.c_double()
        r = self.lib.or_dm_expectation(_c(np.ascontiguousarray(rho.reshape(-1))), int(np.log2(rho.shape[0])),
                                       letters.encode(), coeff, C.byref(out))
        if r != 0:
            raise ValueError("non-real residue")
        return out.value

    def dm_probabilities(self, rho):
        n = int(np.log2(rho.shape[0]))
        out = np.zeros(1 << n)
        self.lib.or_dm_probabilities(_c(np.ascontiguousarray(rho.reshape(-1))), n, _d(out))
        return out

    # --- noise
    def depolarizing(self, p, arity=1):
        out = np.zeros(16 * 16, dtype=np.complex128)
        k = self.lib.or_depolarizing(p, arity, _c(out))
        d = 1 << arity
        return out[: k * d * d].reshape(k, d, d)

    def thermal_relaxation(self, t1, t2, ns):
        out = np.zeros(16, dtype=np.complex128)
        k = self.lib.or_thermal_relaxation(t1, t2, ns, _c(out))
        return out[: k * 4].reshape(k, 2, 2)

    def amplitude_damping(self, g):
        out = np.zeros(8, dtype=np.complex128)
        k = self.lib.or_amplitude_damping(g, _c(out))
        return out[: k * 4].reshape(k, 2, 2)

    def readout_apply_dist(self, dist, p01, p10):
        d = np.ascontiguousarray(dist, dtype=np.float64)
        a = np.ascontiguousarray(p01, dtype=np.float64)
        b = np.ascontiguousarray(p10, dtype=np.float64)
        out = np.zeros_like(d)
        if self.lib.or_readout_apply_dist(_d(d), int(np.log2(len(d))), _d(a), _d(b), _d(out)) != 0:
            raise ValueError("distribution does not sum to 1")
        return out


class Ref:
    """The reference engine compiled from its own sources (oracle/_ref)."""

    @staticmethod
    def available(path: str = REF_PATH) -> bool:
        return os.path.exists(path)

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (build in the container that has /root/reference)")
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p
        self.lib.ref_derive_seed.restype = C.c_uint64
        self.lib.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]

    def _chk(self, r):
        if r != 0:
            raise RuntimeError(f"reference error {r}: {self.lib.ref_last_error().decode()}")

    def set_threads(self, t: int) -> int:
        return self.lib.ref_set_threads(t)

    _OBJ = C.CFUNCTYPE(C.c_double, C.POINTER(C.c_double), C.c_int, C.c_void_p)

    def minimize(self, f, x0, max_evals=500, x_tol=1e-8, f_tol=1e-10, initial_step=1.0):
        """proj/src/neldermead.cpp on a Python objective: (trace, best_x, best_f, converged)."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        n = len(x0)
        cb = self._OBJ(lambda p, k, _ctx: float(f([p[i] for i in range(k)])))
        trace = np.zeros(max_evals)
        best = np.zeros(n)
        evals, conv, bf = C.c_int(), C.c_int(), C.c_double()
        self._chk(self.lib.ref_minimize(cb, None, x0.ctypes.data_as(_dp), n, max_evals, C.c_double(x_tol),
                                        C.c_double(f_tol), C.c_double(initial_step), trace.ctypes.data_as(_dp),
                                        C.byref(evals), best.ctypes.data_as(_dp), C.byref(bf), C.byref(conv)))
        return trace[: evals.value].copy(), best, bf.value, bool(conv.value)

    def rng_u64(self, seed, count):
        out = np.zeros(count, dtype=np.uint64)
        self.lib.ref_rng_u64(C.c_uint64(seed), count, out.ctypes.data_as(_u64p))
        return out

    def random_circuit(self, seed, n, depth, max_arity=3) -> np.ndarray:
        out = np.zeros(depth, dtype=OP_DTYPE)
        self._chk(self.lib.ref_random_circuit(C.c_uint64(seed), n, depth, max_arity, out.ctypes.data))
        return out

    def sv_run(self, n, ops) -> np.ndarray:
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        out = np.zeros(1 << n, dtype=np.complex128)
        self._chk(self.lib.ref_sv_run(n, arr.ctypes.data, C.c_int64(len(arr)), _c(out)))
        return out

    def sv_expectations(self, n, ops, terms):
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        letters = "".join(t[0] for t in terms).encode()
        coeff = np.array([t[1] for t in terms], dtype=np.float64)
        out = np.zeros(len(terms))
        self._chk(self.lib.ref_sv_expectations(n, arr.ctypes.data, C.c_int64(len(arr)), letters, _d(coeff),
                                               len(terms), _d(out)))
        return out

    def sv_sample(self, n, ops, shots, seed):
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        out = np.zeros(1 << n, dtype=np.uint64)
        self._chk(self.lib.ref_sv_sample(n, arr.ctypes.data, C.c_int64(len(arr)), C.c_uint64(shots),
                                         C.c_uint64(seed), out.ctypes.data_as(_u64p)))
        return out

    def sample_distribution(self, dist, shots, seed):
        d = np.ascontiguousarray(dist, dtype=np.float64)
        out = np.zeros(len(d), dtype=np.uint64)
        self._chk(self.lib.ref_sample_distribution(_d(d), int(np.log2(len(d))), C.c_uint64(shots), C.c_uint64(seed),
                                                   out.ctypes.data_as(_u64p)))
        return out

    def dm_run(self, n, ops):
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        out = np.zeros(1 << (2 * n), dtype=np.complex128)
        self._chk(self.lib.ref_dm_run(n, arr.ctypes.data, C.c_int64(len(arr)), _c(out)))
        return out.reshape(1 << n, 1 << n)

    def dm_run_noisy(self, n, ops, noise: NoiseSpec):
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        out = np.zeros(1 << (2 * n), dtype=np.complex128)
        t1, t2, p01, p10 = noise.arrays()
        self._chk(self.lib.ref_dm_run_noisy(n, arr.ctypes.data, C.c_int64(len(arr)), t1, t2, p01, p10,
                                            C.c_double(noise.e1), C.c_double(noise.d1), C.c_double(noise.e2),
                                            C.c_double(noise.d2), _c(out)))
        return out.reshape(1 << n, 1 << n)

    def dm_noisy_reductions(self, n, ops, noise: NoiseSpec, terms):
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        t1, t2, p01, p10 = noise.arrays()
        letters = "".join(t[0] for t in terms).encode()
        coeff = np.array([t[1] for t in terms], dtype=np.float64)
        scal = np.zeros(3)
        ex = np.zeros(len(terms))
        probs = np.zeros(1 << n)
        self._chk(self.lib.ref_dm_noisy_reductions(
            n, arr.ctypes.data, C.c_int64(len(arr)), t1, t2, p01, p10, C.c_double(noise.e1), C.c_double(noise.d1),
            C.c_double(noise.e2), C.c_double(noise.d2), letters, _d(coeff), len(terms), _d(scal), _d(ex), _d(probs)))
        return scal, ex, probs

    def readout_apply_dist(self, dist, p01, p10):
        d = np.ascontiguousarray(dist, dtype=np.float64)
        a = np.ascontiguousarray(p01, dtype=np.float64)
        b = np.ascontiguousarray(p10, dtype=np.float64)
        out = np.zeros_like(d)
        self._chk(self.lib.ref_readout_apply_dist(_d(d), int(np.log2(len(d))), _d(a), _d(b), _d(out)))
        return out

    def sv_time_noreset(self, n, ops, reps):
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        ms = np.zeros(reps)
        ez = C.c_double()
        self._chk(self.lib.ref_sv_time_noreset(n, arr.ctypes.data, C.c_int64(len(arr)), reps, _d(ms), C.byref(ez)))
        return ms, ez.value

    def sv_new(self, n):
        self.lib.ref_sv_new.restype = C.c_void_p
        h = self.lib.ref_sv_new(n)
        if not h:
            raise MemoryError(self.lib.ref_last_error().decode())
        return C.c_void_p(h)

    def sv_free(self, h):
        self.lib.ref_sv_free.argtypes = [C.c_void_p]
        self.lib.ref_sv_free(h)

    def sv_run_timed(self, h, ops) -> float:
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        ms = C.c_double()
        self.lib.ref_sv_run_timed.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, _dp]
        self._chk(self.lib.ref_sv_run_timed(h, arr.ctypes.data, len(arr), C.byref(ms)))
        return ms.value

    def sv_gather(self, h, idx) -> np.ndarray:
        """Amplitudes at the given indices of a persistent reference state."""
        ix = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.zeros(len(ix), dtype=np.complex128)
        self.lib.ref_sv_gather.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        self._chk(self.lib.ref_sv_gather(h, ix.ctypes.data, len(ix), out.ctypes.data))
        return out

    def sv_norm_sq_h(self, h) -> float:
        v = C.c_double()
        self.lib.ref_sv_norm_sq_h.argtypes = [C.c_void_p, _dp]
        self._chk(self.lib.ref_sv_norm_sq_h(h, C.byref(v)))
        return v.value

    def sv_expectations_h(self, h, n, terms) -> np.ndarray:
        letters = "".join(t[0] for t in terms).encode()
        assert all(len(t[0]) == n for t in terms)
        coeff = np.array([t[1] for t in terms], dtype=np.float64)
        out = np.zeros(len(terms))
        self.lib.ref_sv_expectations_h.argtypes = [C.c_void_p, C.c_char_p, _dp, C.c_int, _dp]
        self._chk(self.lib.ref_sv_expectations_h(h, letters, _d(coeff), len(terms), _d(out)))
        return out

    def sv_reset_h(self, h):
        self.lib.ref_sv_reset_h.argtypes = [C.c_void_p]
        self._chk(self.lib.ref_sv_reset_h(h))

    def tfim_sweep(self, calib_json: str, n: int, t_max: float = 3.0, dt: float = 0.1, steps_per_unit: int = 100,
                   max_rows: int = 1000):
        """Reference magnetization sweep rows (no exact column): (t, ideal, noisy, wall ms)."""
        t = np.zeros(max_rows)
        ideal = np.zeros(max_rows)
        noisy = np.zeros(max_rows)
        nrows = C.c_int()
        ms = C.c_double()
        self._chk(self.lib.ref_tfim_sweep(calib_json.encode(), n, C.c_double(t_max), C.c_double(dt), steps_per_unit,
                                          max_rows, _d(t), _d(ideal), _d(noisy), C.byref(nrows), C.byref(ms)))
        k = nrows.value
        return t[:k], ideal[:k], noisy[:k], ms.value

    def traj_time(self, n, ops, noise: NoiseSpec, ntraj, seed):
        """Sequential reference trajectories (shared Rng): (wall ms, <Z0> per trajectory)."""
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        ms = C.c_double()
        z = np.zeros(ntraj)
        t1, t2, p01, p10 = noise.arrays()
        self._chk(self.lib.ref_traj_time(n, arr.ctypes.data, C.c_int64(len(arr)), t1, t2, p01, p10,
                                         C.c_double(noise.e1), C.c_double(noise.d1), C.c_double(noise.e2),
                                         C.c_double(noise.d2), C.c_int64(ntraj), C.c_uint64(seed), C.byref(ms),
                                         _d(z)))
        return ms.value, z

    def dm_time_noisy(self, n, ops, noise: NoiseSpec, reps):
        arr = ops if isinstance(ops, np.ndarray) else list_to_ops(ops)
        ms = np.zeros(reps)
        t1, t2, p01, p10 = noise.arrays()
        self._chk(self.lib.ref_dm_time_noisy(n, arr.ctypes.data, C.c_int64(len(arr)), t1, t2, p01, p10,
                                             C.c_double(noise.e1), C.c_double(noise.d1), C.c_double(noise.e2),
                                             C.c_double(noise.d2), reps, _d(ms)))
        return ms


def qft_closed_form(n: int, ys, prep_seed: int = 7) -> np.ndarray:
    """Closed form of the C2 QFT workload (paper_2401_06861_b200/workloads.qft):
    RY(theta_q) then RZ(phi_q) on every qubit of |0..0> (angles
    Rng(prep_seed).uniform(-pi, pi), ry before rz per qubit), then the QFT in
    the reference gate set with the final swaps.  The prep state is a product
    psi(x) = prod_q psi_q(x_q) with psi_q = (cos(t/2) e^{-i p/2}, sin(t/2) e^{i p/2})
    (proj/src/gates.cpp:61-106), so with x = sum_q x_q 2^q
        out[y] = 2^{-n/2} sum_x psi(x) e^{2 pi i x y / 2^n}
               = 2^{-n/2} prod_q (psi_q(0) + psi_q(1) e^{2 pi i (2^q y mod 2^n) / 2^n}),
    O(n) per amplitude at any n (the reference's 2^n engine needs ~6 min for
    the 2,220 ops at n = 30).  Pinned against oracle/_ref by
    tests/test_scale_parity_cpu.py."""
    u = Port().rng_double(prep_seed, 2 * n)
    psi = []
    for q in range(n):
        th = -np.pi + 2 * np.pi * u[2 * q]
        ph = -np.pi + 2 * np.pi * u[2 * q + 1]
        psi.append((np.cos(th / 2) * np.exp(-0.5j * ph), np.sin(th / 2) * np.exp(0.5j * ph)))
    ys = np.asarray(ys, dtype=np.int64)
    N = 1 << n
    acc = np.full(len(ys), 2.0 ** (-n / 2), dtype=np.complex128)
    for q in range(n):
        frac = ((ys << q) & (N - 1)).astype(np.float64) / N
        acc *= psi[q][0] + psi[q][1] * np.exp(2j * np.pi * frac)
    return acc
