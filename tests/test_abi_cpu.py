"""CPU-side checks of the drop-in boundary (no GPU needed).

* the C-ABI library loads and exports every function include/naqs_b200.h declares;
* the ctypes binding declares the same set;
* contract errors that need no device are raised with the reference's wording;
* the Python surface (naqs._core mirror) imports and builds circuits;
* the synthetic-circuit generator equals the reference's seeded generator.
"""
import os
import re

import numpy as np
import pytest

from paper_2401_06861_b200 import abi, workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "naqs_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nq_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 45
    for name in names:
        assert hasattr(abi.lib, name), name


def test_ctypes_binding_covers_the_header():
    assert set(declared_functions()) == set(abi.SIGNATURES)


def test_abi_version_and_struct_layouts():
    assert abi.lib.nq_abi_version() == 1
    assert abi.OP_DTYPE.itemsize == 48 and abi.SCHED_DTYPE.itemsize == 64


def test_contract_errors_without_a_device():
    with pytest.raises(abi.ContractError, match="qubit count must be in"):
        abi.SV(31)
    with pytest.raises(abi.ContractError, match="qubit count must be in"):
        abi.DM(15)
    with pytest.raises(abi.ContractError):
        abi.SV(0)


def test_python_surface_imports_and_validates():
    from paper_2401_06861_b200 import naqs

    c = naqs.Circuit(3, "t")
    c.add("h", [0]).add("cx", [0, 2]).add("rz", [1], [0.5])
    assert len(c) == 3 and c.num_qubits == 3
    assert c.ops()[1] == ("cx", [0, 2], [])
    with pytest.raises(naqs.NaqsError, match="out of range"):
        c.add("x", [3])
    with pytest.raises(naqs.NaqsError, match="expects 1 parameter"):
        c.add("rx", [0])
    inv = c.inverse()
    assert inv.ops()[0] == ("rz", [1], [-0.5])
    model = naqs.DeviceNoiseModel.zero_noise(4)
    assert model.num_qubits == 4
    m = naqs.load_calibration('{"qubits": [{"t1_us": 10, "t2_us": 20, "readout_p01": 0, "readout_p10": 0}]}')
    assert m.warnings and "clamped" in m.warnings[0]
    with pytest.raises(naqs.NaqsError, match="missing field 'qubits'"):
        naqs.load_calibration("{}")


def test_workload_generator_matches_reference_generator(port):
    from oracle import ops_to_list

    for seed, n, d, ma in [(2024, 30, 200, 3), (17, 3, 12, 3), (4074, 34, 200, 3), (5, 6, 80, 2)]:
        a = [(k, list(q), [float(x) for x in p]) for k, q, p in workloads.random_circuit(seed, n, d, ma)]
        assert a == ops_to_list(port.random_circuit(seed, n, d, ma))


def test_workload_shapes():
    assert len(workloads.qft(30)) == 2 * 30 + 30 + 5 * 435 + 15
    assert len(workloads.vqe_ansatz(28, 3, workloads.vqe_initial_params(28, 3))) == 193
    assert len(workloads.tfim_hamiltonian(28)) == 55
    # ceil(t * spu) steps; 13 ops per step at n = 4 (tests/test_tfim.cpp:57-59)
    assert len(workloads.tfim_trotter(4, 0.5)) == 50 * 13
    assert len(workloads.tfim_trotter(4, 0.0)) == 0


def test_pass_kernels_compile_with_nvrtc_including_exchange_stores():
    """Every pass of a random-circuit plan specialises to source NVRTC accepts
    for sm_100a, in both the in-place form and the exchange-store form a
    sharded flush fuses with a global-qubit swap (out-of-place stores, the
    moved half to the partner's buffer)."""
    ops = workloads.random_circuit(2024, 24, 120)
    for idx in range(2):
        src, ok = abi.jit_debug(24, ops, idx)
        assert ok == 1, src[-2000:]
        assert "xout_r" not in src.split("{", 1)[1]  # in-place pass: no exchange stores
        xsrc, xok = abi.jit_debug(24, ops, idx, xstore=True)
        assert xok == 1, xsrc[-2000:]
        assert "xout_r + (o ^ xmask)" in xsrc and "rr = " in xsrc


def test_dlpack_capsule_lifecycle_without_a_device():
    """The DLPack export path without touching device memory:
    an unconsumed capsule releases its managed tensor when it dies, and a
    consumed one ("used_dltensor", as torch / CuPy rename it) is released by
    the consumer calling the tensor's deleter exactly once."""
    import ctypes as C
    import gc

    view = abi.DeviceArray(0x1000, (8,), "<c16", 0)
    for _ in range(3):  # unconsumed: the capsule destructor frees it
        cap = view.__dlpack__()
        assert len(abi._dl_live) == 1
        del cap
        gc.collect()
        assert len(abi._dl_live) == 0
    cap = view.__dlpack__()
    get = C.pythonapi.PyCapsule_GetPointer
    get.restype, get.argtypes = C.c_void_p, [C.py_object, C.c_char_p]
    ptr = get(cap, b"dltensor")
    mt = abi._DLManagedTensor.from_address(ptr)
    assert mt.dl_tensor.data == 0x1000 and mt.dl_tensor.ndim == 1 and mt.dl_tensor.shape[0] == 8
    assert (mt.dl_tensor.dtype.code, mt.dl_tensor.dtype.bits) == (5, 128)
    rename = C.pythonapi.PyCapsule_SetName
    rename.restype, rename.argtypes = C.c_int, [C.py_object, C.c_char_p]
    used = C.c_char_p(b"used_dltensor")
    assert rename(cap, used) == 0
    del cap
    gc.collect()
    assert len(abi._dl_live) == 1  # consumed: the consumer owns it now
    mt.deleter(ptr)
    assert len(abi._dl_live) == 0
