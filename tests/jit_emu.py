"""Host emulation of the pass kernels the JIT generates (test infrastructure).

The planner's passes (nq_plan_debug) and the generator's sources for them
(nq_jit_debug) are compiled with g++ against pass_ops.cuh built with NQ_EMU
(tests/jit_emu/jit_emu.hpp: CUDA built-ins on std::threads), then run pass by
pass on a host state vector.  This checks the code generator -- register
layouts, relayouts, swizzles, relabelled stores, pending permutations, phase
accumulators, entry-class specialisation -- against the oracle without a GPU.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import re
import subprocess
import tempfile

import numpy as np

from paper_2401_06861_b200 import abi, plan_format

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2401_06861_b200", "csrc")
EMU = os.path.join(ROOT, "tests", "jit_emu")
_CACHE = os.path.join(tempfile.gettempdir(), "nq_jit_emu")
# "address" / "thread": build the emulated kernels with that g++ sanitizer (the
# process must preload its runtime; tests/test_jit_emu_cpu.py runs a child)
SANITIZE = os.environ.get("NQ_EMU_SANITIZE", "")


def sources(n: int, ops: np.ndarray, tile: int, count: int, zterms: bool = False):
    """Generated pass sources; with `zterms` the last one carries the fused
    Z-term epilogue of jit_debug (physical masks: bit 0, bit n-1, bits 0+1)."""
    out = []
    for i in range(count):
        src, _ = abi.jit_debug(n, ops, i, tile_qubits=tile, compile=False, zterms=zterms and i == count - 1)
        out.append(src.split("/* NVRTC LOG")[0])
    return out


def build(srcs) -> C.CDLL:
    os.makedirs(_CACHE, exist_ok=True)
    body = [open(os.path.join(EMU, "emu_main.cpp")).read()]
    for i, s in enumerate(srcs):
        s = s.replace('#include "pass_ops.cuh"', "")
        s = s.replace("extern __shared__ __align__(16) unsigned char smem[];", "unsigned char* const smem = emu_smem;")
        if "double* __restrict__ epart" in s:
            # epilogue kernel: called through a wrapper with the emulator's
            # partial-sum buffer as its extra parameter
            s = re.sub(r"\bnqjit\(", f"nqjit_{i}_ep(", s, count=1)
            s += (f"\nvoid nqjit_{i}(double2* st, const double2* gp, unsigned long long rb, long long nt, double2* xl,"
                  f" double2* xr, unsigned long long xm, unsigned long long xv, int xrot) {{"
                  f" nqjit_{i}_ep(st, gp, rb, nt, xl, xr, xm, xv, xrot, emu_epart); }}\n")
        else:
            s = re.sub(r"\bnqjit\(", f"nqjit_{i}(", s, count=1)
        body.append(s)
    body.append("emu_kernel emu_table[] = {" + ", ".join(f"nqjit_{i}" for i in range(len(srcs))) + "};\n")
    code = "\n".join(body)
    san = ["-fsanitize=" + SANITIZE, "-fno-omit-frame-pointer", "-g"] if SANITIZE else []
    key = hashlib.sha1((code + open(os.path.join(CSRC, "pass_ops.cuh")).read() + " ".join(san)).encode()
                       ).hexdigest()[:16]
    so = os.path.join(_CACHE, f"emu_{key}.so")
    if not os.path.exists(so):
        cpp = so[:-3] + ".cpp"
        with open(cpp, "w") as f:
            f.write(code)
        subprocess.run(["g++", "-std=c++20", "-O1", "-shared", "-fPIC", "-pthread", "-Wno-unknown-pragmas",
                        "-DNQ_EMU", *san, "-I", CSRC, "-I", EMU, "-o", so + ".tmp", cpp], check=True)
        os.replace(so + ".tmp", so)
    lib = C.CDLL(so)
    lib.emu_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_longlong, C.c_int, C.c_longlong]
    lib.emu_set_epart.argtypes = [C.c_void_p]
    return lib


def run(n: int, ops, tile: int, state: np.ndarray | None = None, zterms: bool = False):
    """Apply `ops` (nq_op records or tuples) to `state` (default |0..0>) by
    emulating the generated kernel of every planned pass; returns the state in
    logical (reference) order.  With `zterms` the last pass also runs the
    fused Z-term epilogue (physical masks bit 0, bit n-1, bits 0+1) and the
    result is (state, epilogue sums, final physical-order state)."""
    arr = ops if isinstance(ops, np.ndarray) else abi.make_ops(ops)
    passes = plan_format.decode(abi.plan_debug(n, arr, tile_qubits=tile, relabel=True))
    srcs = sources(n, arr, tile, len(passes), zterms=zterms)
    assert len(srcs) == len(passes), (len(srcs), len(passes))
    lib = build(srcs)
    part = np.zeros(64, dtype=np.float64)
    lib.emu_set_epart(part.ctypes.data)
    st = np.zeros(1 << n, dtype=np.complex128) if state is None else np.array(state, dtype=np.complex128)
    if state is None:
        st[0] = 1.0
    l2p = list(range(n))
    for i, p in enumerate(passes):
        e = 1 << p.ops[0].k
        threads = (1 << p.m) // e
        ntiles = 1 << (n - p.m)
        pool = np.ascontiguousarray(p.pool, dtype=np.complex128)
        smem = (1 << p.m) * 16 + len(pool) * 16  # as jit_launch sizes it
        lib.emu_run(i, st.ctypes.data, pool.ctypes.data, ntiles, threads, smem)
        qst = p.qst if p.qst else p.q
        lab = p.lab if p.lab else list(range(p.m))
        # the logical qubit at load bit q[lab[i]] ends at store bit qst[i]
        move = {p.q[lab[i]]: qst[i] for i in range(p.m)}
        l2p = [move.get(x, x) for x in l2p]
    idx = np.arange(1 << n, dtype=np.int64)
    phys = np.zeros_like(idx)
    for x in range(n):
        phys |= ((idx >> x) & 1) << l2p[x]
    if zterms:
        return st[phys], part[:3].copy(), st
    return st[phys]
