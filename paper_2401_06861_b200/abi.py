"""ctypes binding of the C ABI (include/naqs_b200.h).

This is the reference-side binding a Python host would add:
plain pointers and sizes, no torch types.  The library is the in-tree
``libnaqs_b200.so`` built by ``__graft_entry__.build()``; importing this module
fails loudly when it is missing -- there is no fallback implementation.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnaqs_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA core first (python -c 'import __graft_entry__ as g; g.build()')"
    )

def _torch_nccl():
    """torch's bundled libnccl.so.2, found without importing torch."""
    import importlib.util

    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for d in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    return None


# NCCL is bound lazily by the library (csrc/shard.cpp); prefer torch's copy so
# that importing torch later in the same process still works.
if "NQ_NCCL_LIB" not in os.environ and _torch_nccl():
    os.environ["NQ_NCCL_LIB"] = _torch_nccl()

lib = C.CDLL(LIB_PATH)

# Gate kinds: ordinals of naqs::GateKind (proj/include/naqs/circuit.hpp:15-37).
KINDS = [
    "x", "y", "z", "h", "s", "sdg", "t", "tdg", "id",
    "rx", "ry", "rz", "u1", "u2", "u3",
    "cx", "cz", "swap", "ccx", "measure", "barrier",
]
KIND = {k: i for i, k in enumerate(KINDS)}
ARITY = {k: (2 if k in ("cx", "cz", "swap") else 3 if k == "ccx" else 1) for k in KINDS}
NPARAMS = {k: (1 if k in ("rx", "ry", "rz", "u1") else 2 if k == "u2" else 3 if k == "u3" else 0) for k in KINDS}

OP_DTYPE = np.dtype(
    [("kind", "<i4"), ("nqubits", "<i4"), ("qubits", "<i4", (3,)), ("reserved", "<i4"), ("params", "<f8", (3,))],
    align=True,
)
assert OP_DTYPE.itemsize == 48
SCHED_DTYPE = np.dtype(
    [("type", "<i4"), ("nkraus", "<i4"), ("kraus_offset", "<i8"), ("op", OP_DTYPE)], align=True
)
assert SCHED_DTYPE.itemsize == 64


class nq_profile(C.Structure):
    _fields_ = [("region_ms", C.c_double), ("pass_ms", C.c_double), ("pass_launches", C.c_int64),
                ("pass_bytes", C.c_double), ("kernel_launches", C.c_int64), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64)]


class nq_opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("max_qubits", C.c_int32), ("tile_qubits", C.c_int32), ("fuse", C.c_int32)]


NQ_OK, NQ_ERR_CONTRACT = 0, 1


class NaqsError(RuntimeError):
    """Any non-OK status (naqs::Error)."""


class ContractError(NaqsError):
    """NQ_ERR_CONTRACT (naqs::ContractError)."""


_p = C.c_void_p
_pp = C.POINTER(C.c_void_p)
_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_ucp = C.POINTER(C.c_ubyte)

# name -> argtypes (restype is nq_status = int for all but the first two)
SIGNATURES = {
    "nq_last_error": ([], C.c_char_p),
    "nq_abi_version": ([], C.c_int),
    "nq_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "nq_default_opts": ([C.POINTER(nq_opts)], C.c_int),
    "nq_sv_create": ([C.c_int, C.POINTER(nq_opts), _pp], C.c_int),
    "nq_sv_destroy": ([_p], C.c_int),
    "nq_sv_clone": ([_p, _pp], C.c_int),
    "nq_sv_reset": ([_p], C.c_int),
    "nq_sv_num_qubits": ([_p, C.POINTER(C.c_int)], C.c_int),
    "nq_sv_apply_ops": ([_p, _p, C.c_int64], C.c_int),
    "nq_sv_apply_matrix": ([_p, _i32p, C.c_int, _dp], C.c_int),
    "nq_sv_scale": ([_p, C.c_double], C.c_int),
    "nq_sv_flush": ([_p], C.c_int),
    "nq_sv_norm_sq": ([_p, _dp], C.c_int),
    "nq_sv_expectation_batch": ([_p, _u64p, _u64p, _i32p, _dp, C.c_int, _dp], C.c_int),
    "nq_sv_probabilities": ([_p, _dp], C.c_int),
    "nq_sv_sample_sorted": ([_p, _dp, C.c_uint64, _u64p, _u64p, _u64p], C.c_int),
    "nq_sv_kraus_weights": ([_p, _i32p, C.c_int, C.c_int, _dp, _dp], C.c_int),
    "nq_sv_get_amplitudes": ([_p, C.c_uint64, C.c_uint64, _dp], C.c_int),
    "nq_sv_set_amplitudes": ([_p, C.c_uint64, C.c_uint64, _dp], C.c_int),
    "nq_sv_device_ptr": ([_p, _pp], C.c_int),
    "nq_sv_device": ([_p, C.POINTER(C.c_int)], C.c_int),
    "nq_sv_probabilities_device": ([_p, C.POINTER(_dp)], C.c_int),
    "nq_sv_local_range": ([_p, _u64p, _u64p], C.c_int),
    "nq_sv_last_stats": ([_p, _i64p, _i64p, _i64p, _i64p], C.c_int),
    "nq_sv_synchronize": ([_p], C.c_int),
    "nq_dm_create": ([C.c_int, C.POINTER(nq_opts), _pp], C.c_int),
    "nq_dm_destroy": ([_p], C.c_int),
    "nq_dm_clone": ([_p, _pp], C.c_int),
    "nq_dm_reset": ([_p], C.c_int),
    "nq_dm_num_qubits": ([_p, C.POINTER(C.c_int)], C.c_int),
    "nq_dm_apply_ops": ([_p, _p, C.c_int64], C.c_int),
    "nq_dm_apply_channel": ([_p, _i32p, C.c_int, C.c_int, _dp], C.c_int),
    "nq_dm_apply_schedule": ([_p, _p, C.c_int64, _dp], C.c_int),
    "nq_dm_flush": ([_p], C.c_int),
    "nq_dm_trace": ([_p, _dp], C.c_int),
    "nq_dm_purity": ([_p, _dp], C.c_int),
    "nq_dm_hermiticity_residual": ([_p, _dp], C.c_int),
    "nq_dm_expectation_batch": ([_p, _u64p, _u64p, _i32p, _dp, C.c_int, _dp, _dp], C.c_int),
    "nq_dm_probabilities": ([_p, _dp], C.c_int),
    "nq_dm_device_ptr": ([_p, _pp], C.c_int),
    "nq_dm_device": ([_p, C.POINTER(C.c_int)], C.c_int),
    "nq_dm_probabilities_device": ([_p, C.POINTER(_dp)], C.c_int),
    "nq_dm_get_entries": ([_p, C.c_uint64, C.c_uint64, _dp], C.c_int),
    "nq_dm_set_entries": ([_p, C.c_uint64, C.c_uint64, _dp], C.c_int),
    "nq_dm_last_stats": ([_p, _i64p, _i64p, _i64p, _i64p], C.c_int),
    "nq_dm_synchronize": ([_p], C.c_int),
    "nq_readout_apply_dist": ([_dp, C.c_int, _dp, _dp, _dp], C.c_int),
    "nq_sample_dist_sorted": ([_dp, C.c_uint64, _dp, C.c_uint64, _u64p, _u64p, _u64p], C.c_int),
    "nq_comm_unique_id": ([_ucp], C.c_int),
    "nq_sv_create_sharded": ([C.c_int, C.c_int, C.c_int, _ucp, C.POINTER(nq_opts), _pp], C.c_int),
    "nq_sv_comm_stats": ([_p, _i64p, _i64p], C.c_int),
    "nq_sv_comm_fused": ([_p, _i64p, C.POINTER(C.c_int)], C.c_int),
    "nq_shard_debug": ([C.c_int, C.c_int, _p, C.c_int64, C.c_int, _i64p, C.c_int64, _i64p], C.c_int),
    "nq_profile_begin": ([C.c_int, C.c_int], C.c_int),
    "nq_profile_end": ([C.c_int, C.POINTER(nq_profile)], C.c_int),
    "nq_jit_wait": ([], C.c_int),
    "nq_jit_shutdown": ([], C.c_int),
    "nq_batch_run": ([C.c_int, C.c_int, C.c_int64, _p, _p, _dp, _p, _p, _p, _p, C.c_int, _p, _p, _p, C.c_int],
                     C.c_int),
    "nq_traj_run": ([C.c_int, _p, C.c_int64, _dp, C.c_int64, _p, _p, _p, _p, _p, C.c_int, _p, _p, _dp, C.c_int],
                    C.c_int),
    "nq_jit_stats": ([_i64p, _i64p, _i64p, _i64p], C.c_int),
    "nq_jit_debug": ([C.c_int, _p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int64, _i64p,
                      C.POINTER(C.c_int)], C.c_int),
    "nq_plan_debug": ([C.c_int, _p, C.c_int64, C.c_int, C.c_int, _ucp, C.c_int64, _i64p], C.c_int),
}

for _name, (_args, _res) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res

# Run-time kernel compilations still in flight at interpreter exit are
# cancelled / awaited before native teardown starts.
atexit.register(lib.nq_jit_shutdown)


def check(status: int) -> None:
    if status == NQ_OK:
        return
    msg = lib.nq_last_error().decode()
    if status == NQ_ERR_CONTRACT:
        raise ContractError(msg)
    raise NaqsError(f"status {status}: {msg}")


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def make_ops(ops: Iterable[Sequence]) -> np.ndarray:
    """[(name, qubits, params), ...] -> packed nq_op array."""
    ops = list(ops)
    arr = np.zeros(len(ops), dtype=OP_DTYPE)
    for i, op in enumerate(ops):
        name, qubits = op[0], op[1]
        params = op[2] if len(op) > 2 else ()
        arr[i]["kind"] = KIND[name]
        arr[i]["nqubits"] = len(qubits)
        for j, q in enumerate(qubits):
            arr[i]["qubits"][j] = q
        for j, p in enumerate(params):
            arr[i]["params"][j] = p
    return arr


def opts(device: int = -1, max_qubits: int = 0, tile_qubits: int = 0, fuse: bool = True) -> nq_opts:
    o = nq_opts()
    check(lib.nq_default_opts(C.byref(o)))
    o.device, o.max_qubits, o.tile_qubits, o.fuse = device, max_qubits, tile_qubits, 1 if fuse else 0
    return o


def pauli_masks(letters: str):
    flip = signs = ny = 0
    for i, L in enumerate(letters):
        if L in "XY":
            flip |= 1 << i
        if L in "YZ":
            signs |= 1 << i
        if L == "Y":
            ny += 1
    return flip, signs, ny


class SV:
    """Thin owner of an nq_sv handle (C ABI)."""

    def __init__(self, n: int, *, handle=None, **kw):
        self.n = n
        if handle is not None:
            self.h = handle
        else:
            self.h = C.c_void_p()
            check(lib.nq_sv_create(n, C.byref(opts(**kw)), C.byref(self.h)))

    def close(self):
        if self.h:
            check(lib.nq_sv_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def clone(self) -> "SV":
        h = C.c_void_p()
        check(lib.nq_sv_clone(self.h, C.byref(h)))
        return SV(self.n, handle=h)

    def reset(self):
        check(lib.nq_sv_reset(self.h))

    def apply(self, ops) -> "SV":
        arr = ops if isinstance(ops, np.ndarray) else make_ops(ops)
        check(lib.nq_sv_apply_ops(self.h, arr.ctypes.data, len(arr)))
        return self

    def apply_matrix(self, qubits, mat):
        q = np.asarray(qubits, dtype=np.int32)
        m = np.ascontiguousarray(np.asarray(mat, dtype=np.complex128))
        check(lib.nq_sv_apply_matrix(self.h, _ptr(q, C.c_int32), len(q), m.view(np.float64).ctypes.data_as(_dp)))

    def scale(self, f: float):
        check(lib.nq_sv_scale(self.h, f))

    def flush(self):
        check(lib.nq_sv_flush(self.h))

    def synchronize(self):
        check(lib.nq_sv_synchronize(self.h))

    def amplitudes(self, offset: int = 0, count: int | None = None) -> np.ndarray:
        count = (1 << self.n) - offset if count is None else count
        out = np.empty(count, dtype=np.complex128)
        check(lib.nq_sv_get_amplitudes(self.h, offset, count, out.view(np.float64).ctypes.data_as(_dp)))
        return out

    def _device(self) -> int:
        d = C.c_int()
        check(lib.nq_sv_device(self.h, C.byref(d)))
        return d.value

    def device_view(self) -> DeviceArray:
        """Zero-copy view of the (flushed) amplitudes in HBM:
        complex128, 2^n (a sharded state: this rank's 2^nloc block, global
        offset in ``.offset``).  The state's queued work is synchronised first."""
        p = C.c_void_p()
        check(lib.nq_sv_device_ptr(self.h, C.byref(p)))
        check(lib.nq_sv_synchronize(self.h))
        off, cnt = C.c_uint64(), C.c_uint64()
        check(lib.nq_sv_local_range(self.h, C.byref(off), C.byref(cnt)))
        return DeviceArray(p.value, (cnt.value,), "<c16", self._device(), self, off.value)

    def device_probabilities(self) -> DeviceArray:
        """|a_i|^2 on the device (no 2^n host copy), float64, in a buffer owned
        by the state: valid until the state is next modified."""
        p = C.POINTER(C.c_double)()
        check(lib.nq_sv_probabilities_device(self.h, C.byref(p)))
        off, cnt = C.c_uint64(), C.c_uint64()
        check(lib.nq_sv_local_range(self.h, C.byref(off), C.byref(cnt)))
        return DeviceArray(C.cast(p, C.c_void_p).value, (cnt.value,), "<f8", self._device(), self, off.value)

    def local_count(self) -> int:
        return 1 << self.n if getattr(self, "world", 1) == 1 else 1 << (self.n - (self.world.bit_length() - 1))

    def set_amplitudes(self, amps, offset: int = 0):
        a = np.ascontiguousarray(np.asarray(amps, dtype=np.complex128))
        check(lib.nq_sv_set_amplitudes(self.h, offset, len(a), a.view(np.float64).ctypes.data_as(_dp)))

    def norm_sq(self) -> float:
        v = C.c_double()
        check(lib.nq_sv_norm_sq(self.h, C.byref(v)))
        return v.value

    def expectations(self, terms) -> np.ndarray:
        """terms: [(letters, coeff), ...] with letters[i] acting on qubit i."""
        flip = np.array([pauli_masks(t[0])[0] for t in terms], dtype=np.uint64)
        signs = np.array([pauli_masks(t[0])[1] for t in terms], dtype=np.uint64)
        ny = np.array([pauli_masks(t[0])[2] for t in terms], dtype=np.int32)
        coeff = np.array([t[1] for t in terms], dtype=np.float64)
        out = np.zeros(len(terms))
        check(lib.nq_sv_expectation_batch(self.h, _ptr(flip, C.c_uint64), _ptr(signs, C.c_uint64),
                                          _ptr(ny, C.c_int32), _ptr(coeff, C.c_double), len(terms),
                                          _ptr(out, C.c_double)))
        return out

    def probabilities(self) -> np.ndarray:
        out = np.empty(1 << self.n)
        check(lib.nq_sv_probabilities(self.h, _ptr(out, C.c_double)))
        return out

    def sample_sorted(self, sorted_u: np.ndarray):
        u = np.ascontiguousarray(sorted_u, dtype=np.float64)
        idx = np.zeros(max(len(u), 1), dtype=np.uint64)
        cnt = np.zeros(max(len(u), 1), dtype=np.uint64)
        k = C.c_uint64()
        check(lib.nq_sv_sample_sorted(self.h, _ptr(u, C.c_double), len(u), _ptr(idx, C.c_uint64),
                                      _ptr(cnt, C.c_uint64), C.byref(k)))
        return idx[: k.value].copy(), cnt[: k.value].copy()

    def kraus_weights(self, qubits, kraus) -> np.ndarray:
        q = np.asarray(qubits, dtype=np.int32)
        ks = np.ascontiguousarray(np.asarray(kraus, dtype=np.complex128))
        out = np.zeros(len(ks))
        check(lib.nq_sv_kraus_weights(self.h, _ptr(q, C.c_int32), len(q), len(ks),
                                      ks.view(np.float64).ctypes.data_as(_dp), _ptr(out, C.c_double)))
        return out

    def stats(self):
        v = [C.c_int64() for _ in range(4)]
        check(lib.nq_sv_last_stats(self.h, *[C.byref(x) for x in v]))
        return {"passes": v[0].value, "microops": v[1].value, "source_ops": v[2].value, "launches": v[3].value}

    @classmethod
    def sharded(cls, n: int, rank: int, world: int, uid: bytes, **kw) -> "SV":
        """State of n qubits split over `world` ranks (one GPU each); every rank
        must call this (and every later method) collectively."""
        h = C.c_void_p()
        u = (C.c_ubyte * 128).from_buffer_copy(uid)
        check(lib.nq_sv_create_sharded(n, rank, world, u, C.byref(opts(**kw)), C.byref(h)))
        sv = cls(n, handle=h)
        sv.world = world
        return sv

    def comm_stats(self):
        a, b = C.c_int64(), C.c_int64()
        check(lib.nq_sv_comm_stats(self.h, C.byref(a), C.byref(b)))
        f, alt = C.c_int64(), C.c_int()
        check(lib.nq_sv_comm_fused(self.h, C.byref(f), C.byref(alt)))
        return {"exchanges": a.value, "bytes_sent": b.value, "fused": f.value, "alt_buffer": alt.value == 1,
                "staged": alt.value == 2}


def comm_unique_id() -> bytes:
    u = (C.c_ubyte * 128)()
    check(lib.nq_comm_unique_id(u))
    return bytes(u)


def shard_debug(n: int, world: int, ops, rebalance: bool = True):
    """Host schedule of a sharded flush: list of ("exchange", gbit, vbit) and
    ("segment", [(type, k, bits, ctrl, matrix), ...]) in physical bits."""
    arr = ops if isinstance(ops, np.ndarray) else make_ops(ops)
    size = C.c_int64()
    fl = 1 if rebalance else 0
    check(lib.nq_shard_debug(n, world, arr.ctypes.data, len(arr), fl, None, 0, C.byref(size)))
    buf = np.zeros(max(size.value, 1), dtype=np.int64)
    check(lib.nq_shard_debug(n, world, arr.ctypes.data, len(arr), fl, buf.ctypes.data_as(_i64p), len(buf),
                             C.byref(size)))
    out, i = [], 0
    types = {0: "dense", 1: "diag", 2: "xperm", 3: "swap", 4: "depol", 5: "nop"}
    while i < size.value:
        kind, a, b, cnt = (int(x) for x in buf[i:i + 4])
        i += 4
        if kind == 1:
            out.append(("exchange", a, b))
            continue
        seg = []
        for _ in range(cnt):
            t, k, b0, b1, b2, b3, ctrl, msz = (int(x) for x in buf[i:i + 8])
            i += 8
            mat = buf[i:i + 2 * msz].copy().view(np.float64).reshape(-1, 2)
            i += 2 * msz
            seg.append((types[t], k, [b0, b1, b2, b3][:k], ctrl & ((1 << 64) - 1), mat[:, 0] + 1j * mat[:, 1]))
        out.append(("segment", seg))
    return out


class _DLDevice(C.Structure):
    _fields_ = [("device_type", C.c_int32), ("device_id", C.c_int32)]


class _DLDataType(C.Structure):
    _fields_ = [("code", C.c_uint8), ("bits", C.c_uint8), ("lanes", C.c_uint16)]


class _DLTensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("device", _DLDevice), ("ndim", C.c_int32), ("dtype", _DLDataType),
                ("shape", C.POINTER(C.c_int64)), ("strides", C.POINTER(C.c_int64)), ("byte_offset", C.c_uint64)]


_DLDeleter = C.CFUNCTYPE(None, C.c_void_p)


class _DLManagedTensor(C.Structure):
    _fields_ = [("dl_tensor", _DLTensor), ("manager_ctx", C.c_void_p), ("deleter", _DLDeleter)]


_KDL_CUDA = 2
_DL_CODES = {"<c16": (5, 128), "<f8": (2, 64)}  # kDLComplex / kDLFloat
_dl_live = {}  # manager_ctx -> (managed tensor, shape array, owner): alive until the consumer's deleter


@_DLDeleter
def _dl_delete(ptr):
    mt = _DLManagedTensor.from_address(ptr)
    _dl_live.pop(mt.manager_ctx, None)


# the destructor receives the dying capsule as a raw pointer: wrapping it in a
# py_object would take a new reference to an object at refcount 0 (resurrect
# it) and crash when that reference is dropped
_PyCapsule_Destructor = C.CFUNCTYPE(None, C.c_void_p)
# private prototypes: C.pythonapi caches one function object per symbol and
# other libraries (torch among them) re-declare argtypes on the shared ones
_capsule_new = C.PYFUNCTYPE(C.py_object, C.c_void_p, C.c_char_p, _PyCapsule_Destructor)(
    ("PyCapsule_New", C.pythonapi))
_capsule_is_valid = C.PYFUNCTYPE(C.c_int, C.c_void_p, C.c_char_p)(("PyCapsule_IsValid", C.pythonapi))
_capsule_get_ptr = C.PYFUNCTYPE(C.c_void_p, C.c_void_p, C.c_char_p)(("PyCapsule_GetPointer", C.pythonapi))


@_PyCapsule_Destructor
def _dl_capsule_destructor(cap):
    # never consumed (still named "dltensor"): release it ourselves
    if _capsule_is_valid(cap, b"dltensor"):
        _dl_delete(_capsule_get_ptr(cap, b"dltensor"))


class DeviceArray:
    """Zero-copy view of a device array owned by a state:
    ``__cuda_array_interface__`` (v3) and DLPack (``__dlpack__`` /
    ``__dlpack_device__``), e.g. ``torch.from_dlpack(view)`` or CuPy.  The
    view keeps its owner alive; it is valid until the owner is modified,
    flushed again or closed.  ``offset`` is the global index of element 0
    (a sharded state's rank block starts at rank << n_local)."""

    def __init__(self, ptr: int, shape, typestr: str, device: int, owner=None, offset: int = 0):
        self.ptr, self.shape, self.typestr, self.device = ptr, tuple(shape), typestr, device
        self.owner, self.offset = owner, offset

    @property
    def count(self) -> int:
        c = 1
        for d in self.shape:
            c *= d
        return c

    @property
    def __cuda_array_interface__(self):
        return {"shape": self.shape, "typestr": self.typestr, "data": (self.ptr, False), "version": 3,
                "strides": None, "stream": None}

    def __dlpack_device__(self):
        return (_KDL_CUDA, self.device)

    def __dlpack__(self, stream=None, max_version=None, dl_device=None, copy=None):
        if copy:
            raise BufferError("DeviceArray exports zero-copy views only")
        # the owner's stream was synchronised when the view was made, so any
        # consumer stream may read it without further ordering
        shape = (C.c_int64 * len(self.shape))(*self.shape)
        mt = _DLManagedTensor()
        code, bits = _DL_CODES[self.typestr]
        mt.dl_tensor = _DLTensor(C.c_void_p(self.ptr), _DLDevice(_KDL_CUDA, self.device), len(self.shape),
                                 _DLDataType(code, bits, 1), shape, None, 0)
        key = C.addressof(mt)
        mt.manager_ctx = key
        mt.deleter = _dl_delete
        _dl_live[key] = (mt, shape, self)
        return _capsule_new(key, b"dltensor", _dl_capsule_destructor)


DeviceAmplitudes = DeviceArray  # round-1 name


class DM:
    """Thin owner of an nq_dm handle (C ABI)."""

    def __init__(self, n: int, *, handle=None, **kw):
        self.n = n
        if handle is not None:
            self.h = handle
        else:
            self.h = C.c_void_p()
            check(lib.nq_dm_create(n, C.byref(opts(**kw)), C.byref(self.h)))

    def close(self):
        if self.h:
            check(lib.nq_dm_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def apply(self, ops) -> "DM":
        arr = ops if isinstance(ops, np.ndarray) else make_ops(ops)
        check(lib.nq_dm_apply_ops(self.h, arr.ctypes.data, len(arr)))
        return self

    def apply_channel(self, qubits, kraus):
        q = np.asarray(qubits, dtype=np.int32)
        ks = np.ascontiguousarray(np.asarray(kraus, dtype=np.complex128))
        check(lib.nq_dm_apply_channel(self.h, _ptr(q, C.c_int32), len(q), len(ks),
                                      ks.view(np.float64).ctypes.data_as(_dp)))

    def apply_schedule(self, items):
        """items: [("gate", (name, qubits, params)) | ("channel", qubits, kraus_list)]."""
        arr, p = make_schedule(items)
        check(lib.nq_dm_apply_schedule(self.h, arr.ctypes.data, len(arr), p.view(np.float64).ctypes.data_as(_dp)))

    def flush(self):
        check(lib.nq_dm_flush(self.h))

    def synchronize(self):
        check(lib.nq_dm_synchronize(self.h))

    def rho(self) -> np.ndarray:
        d = 1 << self.n
        out = np.empty(d * d, dtype=np.complex128)
        check(lib.nq_dm_get_entries(self.h, 0, d * d, out.view(np.float64).ctypes.data_as(_dp)))
        return out.reshape(d, d)

    def set_rho(self, rho):
        a = np.ascontiguousarray(np.asarray(rho, dtype=np.complex128).reshape(-1))
        check(lib.nq_dm_set_entries(self.h, 0, len(a), a.view(np.float64).ctypes.data_as(_dp)))

    def _device(self) -> int:
        d = C.c_int()
        check(lib.nq_dm_device(self.h, C.byref(d)))
        return d.value

    def device_view(self) -> DeviceArray:
        """Zero-copy view of row-major rho (2^n x 2^n complex128) in HBM."""
        p = C.c_void_p()
        check(lib.nq_dm_device_ptr(self.h, C.byref(p)))
        d = 1 << self.n
        return DeviceArray(p.value, (d, d), "<c16", self._device(), self)

    def device_probabilities(self) -> DeviceArray:
        p = C.POINTER(C.c_double)()
        check(lib.nq_dm_probabilities_device(self.h, C.byref(p)))
        return DeviceArray(C.cast(p, C.c_void_p).value, (1 << self.n,), "<f8", self._device(), self)

    def _scalar(self, fn) -> float:
        v = C.c_double()
        check(fn(self.h, C.byref(v)))
        return v.value

    def trace(self):
        return self._scalar(lib.nq_dm_trace)

    def purity(self):
        return self._scalar(lib.nq_dm_purity)

    def hermiticity_residual(self):
        return self._scalar(lib.nq_dm_hermiticity_residual)

    def expectations(self, terms):
        flip = np.array([pauli_masks(t[0])[0] for t in terms], dtype=np.uint64)
        signs = np.array([pauli_masks(t[0])[1] for t in terms], dtype=np.uint64)
        ny = np.array([pauli_masks(t[0])[2] for t in terms], dtype=np.int32)
        coeff = np.array([t[1] for t in terms], dtype=np.float64)
        re = np.zeros(len(terms))
        im = np.zeros(len(terms))
        check(lib.nq_dm_expectation_batch(self.h, _ptr(flip, C.c_uint64), _ptr(signs, C.c_uint64),
                                          _ptr(ny, C.c_int32), _ptr(coeff, C.c_double), len(terms),
                                          _ptr(re, C.c_double), _ptr(im, C.c_double)))
        return re, im

    def probabilities(self):
        out = np.empty(1 << self.n)
        check(lib.nq_dm_probabilities(self.h, _ptr(out, C.c_double)))
        return out

    def stats(self):
        v = [C.c_int64() for _ in range(4)]
        check(lib.nq_dm_last_stats(self.h, *[C.byref(x) for x in v]))
        return {"passes": v[0].value, "microops": v[1].value, "source_ops": v[2].value, "launches": v[3].value}


def readout_apply_dist(dist, p01, p10) -> np.ndarray:
    d = np.ascontiguousarray(dist, dtype=np.float64)
    n = int(np.log2(len(d)))
    a = np.ascontiguousarray(p01, dtype=np.float64)
    b = np.ascontiguousarray(p10, dtype=np.float64)
    out = np.empty_like(d)
    check(lib.nq_readout_apply_dist(_ptr(d, C.c_double), n, _ptr(a, C.c_double), _ptr(b, C.c_double),
                                    _ptr(out, C.c_double)))
    return out


def sample_dist_sorted(dist, sorted_u):
    d = np.ascontiguousarray(dist, dtype=np.float64)
    u = np.ascontiguousarray(sorted_u, dtype=np.float64)
    idx = np.zeros(max(len(u), 1), dtype=np.uint64)
    cnt = np.zeros(max(len(u), 1), dtype=np.uint64)
    k = C.c_uint64()
    check(lib.nq_sample_dist_sorted(_ptr(d, C.c_double), len(d), _ptr(u, C.c_double), len(u),
                                    _ptr(idx, C.c_uint64), _ptr(cnt, C.c_uint64), C.byref(k)))
    return idx[: k.value].copy(), cnt[: k.value].copy()


def plan_debug(n: int, ops, tile_qubits: int = 0, fuse: bool = True, relabel: bool = False) -> bytes:
    arr = ops if isinstance(ops, np.ndarray) else make_ops(ops)
    size = C.c_int64()
    flags = (1 if fuse else 0) | (2 if relabel else 0)
    check(lib.nq_plan_debug(n, arr.ctypes.data, len(arr), tile_qubits, flags, None, 0, C.byref(size)))
    buf = (C.c_ubyte * max(size.value, 1))()
    check(lib.nq_plan_debug(n, arr.ctypes.data, len(arr), tile_qubits, flags, buf, size.value, C.byref(size)))
    return bytes(buf)[: size.value]


def profile_begin(device: int = -1, per_pass_events: bool = True) -> None:
    check(lib.nq_profile_begin(device, 1 if per_pass_events else 0))


def profile_end(device: int = -1) -> dict:
    p = nq_profile()
    check(lib.nq_profile_end(device, C.byref(p)))
    return {k: getattr(p, k) for k, _ in nq_profile._fields_}


def jit_wait() -> None:
    check(lib.nq_jit_wait())


def jit_stats() -> dict:
    v = [C.c_int64() for _ in range(4)]
    check(lib.nq_jit_stats(*[C.byref(x) for x in v]))
    return dict(zip(("compiled", "failed", "misses", "launches"), (x.value for x in v)))


def jit_debug(n: int, ops, pass_index: int, tile_qubits: int = 0, compile: bool = True, xstore: bool = False,
              segment: bool = False, staged: str = "", zterms: bool = False):
    """Generated source of one planned pass (and whether NVRTC compiles it):
    as a single-device state plans it, or as a sharded segment (`segment`:
    no relabelling stores); `xstore`: the exchange-store form; `staged`
    ("rest" / "tile": where the exchanged bit lies): the staged form;
    `zterms`: with a fused Z-term expectation epilogue."""
    arr = ops if isinstance(ops, np.ndarray) else make_ops(ops)
    size = C.c_int64()
    ok = C.c_int()
    xs = (2 if xstore else 0) | (4 if segment else 0) | {"": 0, "rest": 8, "tile": 24}[staged] | (32 if zterms else 0)
    check(lib.nq_jit_debug(n, arr.ctypes.data, len(arr), tile_qubits, pass_index, xs, None, 0, C.byref(size),
                           C.byref(ok)))
    buf = C.create_string_buffer(size.value + (1 << 16))
    check(lib.nq_jit_debug(n, arr.ctypes.data, len(arr), tile_qubits, pass_index, (1 if compile else 0) | xs, buf,
                           len(buf), C.byref(size), C.byref(ok)))
    return buf.raw[: size.value].decode(), ok.value


def make_schedule(items):
    """Encode [("gate", (name, qubits, params)) | ("channel", qubits, kraus_list)]
    as (nq_sched_item array, complex Kraus pool)."""
    arr = np.zeros(len(items), dtype=SCHED_DTYPE)
    pool = []
    off = 0
    for i, it in enumerate(items):
        if it[0] == "gate":
            arr[i]["type"] = 0
            arr[i]["op"] = make_ops([it[1]])[0]
        else:
            qubits, kraus = it[1], np.asarray(it[2], dtype=np.complex128)
            arr[i]["type"] = 1
            arr[i]["nkraus"] = len(kraus)
            arr[i]["kraus_offset"] = off
            arr[i]["op"]["nqubits"] = len(qubits)
            for j, q in enumerate(qubits):
                arr[i]["op"]["qubits"][j] = q
            pool.append(kraus.reshape(-1))
            off += kraus.size
    p = np.ascontiguousarray(np.concatenate(pool) if pool else np.zeros(1, dtype=np.complex128))
    return arr, p


def traj_run(n: int, items, ntraj: int, uniforms, terms, branches: bool = False, amplitudes: bool = False,
             device: int = -1):
    """Batched run_trajectory (nq_traj_run): `uniforms` is (ntraj, channels)
    in the order the sequential loop draws them.  Returns (expectations
    [ntraj, nterms], branches [ntraj, C] or None, amplitudes [ntraj, 2^n] or None)."""
    arr, p = make_schedule(items)
    nch = int(np.sum(arr["type"] == 1))
    u = np.ascontiguousarray(np.asarray(uniforms, dtype=np.float64).reshape(ntraj, nch))
    flip = np.array([pauli_masks(t[0])[0] for t in terms], dtype=np.uint64)
    signs = np.array([pauli_masks(t[0])[1] for t in terms], dtype=np.uint64)
    ny = np.array([pauli_masks(t[0])[2] for t in terms], dtype=np.int32)
    coeff = np.array([t[1] for t in terms], dtype=np.float64)
    out = np.zeros((ntraj, len(terms)))
    br = np.zeros((ntraj, nch), dtype=np.int32) if branches else None
    am = np.zeros((ntraj, 1 << n), dtype=np.complex128) if amplitudes else None
    check(lib.nq_traj_run(n, arr.ctypes.data, len(arr), p.view(np.float64).ctypes.data_as(_dp), ntraj,
                          _ptr(u, C.c_double), _ptr(flip, C.c_uint64), _ptr(signs, C.c_uint64),
                          _ptr(ny, C.c_int32), _ptr(coeff, C.c_double), len(terms), _ptr(out, C.c_double),
                          br.ctypes.data_as(C.POINTER(C.c_int32)) if br is not None else None,
                          am.view(np.float64).ctypes.data_as(_dp) if am is not None else None, device))
    return out, br, am


def batch_run(n: int, circuits_items, terms, dm: bool = False, probabilities: bool = False, device: int = -1):
    """nq_batch_run: circuits_items = one schedule item list per circuit (see
    make_schedule).  Returns (expectations [B, T], imaginary residue [B, T],
    probabilities [B, 2^n] or None)."""
    B = len(circuits_items)
    flat, off = [], [0]
    for items in circuits_items:
        flat.extend(items)
        off.append(len(flat))
    arr, p = make_schedule(flat)
    offs = np.array(off, dtype=np.int64)
    flip = np.array([pauli_masks(t[0])[0] for t in terms], dtype=np.uint64)
    signs = np.array([pauli_masks(t[0])[1] for t in terms], dtype=np.uint64)
    ny = np.array([pauli_masks(t[0])[2] for t in terms], dtype=np.int32)
    coeff = np.array([t[1] for t in terms], dtype=np.float64)
    out = np.zeros((B, len(terms)))
    oim = np.zeros((B, len(terms)))
    pr = np.zeros((B, 1 << n)) if probabilities else None
    check(lib.nq_batch_run(n, 1 if dm else 0, B, offs.ctypes.data, arr.ctypes.data,
                           p.view(np.float64).ctypes.data_as(_dp), _ptr(flip, C.c_uint64), _ptr(signs, C.c_uint64),
                           _ptr(ny, C.c_int32), _ptr(coeff, C.c_double), len(terms), _ptr(out, C.c_double),
                           _ptr(oim, C.c_double), pr.ctypes.data if pr is not None else None, device))
    return out, oim, pr


def device_count() -> int:
    n = C.c_int()
    st = lib.nq_device_count(C.byref(n))
    return n.value if st == NQ_OK else 0
