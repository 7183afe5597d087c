"""The pass-kernel generator (csrc/jit.cpp) checked on the host: the
generated sources of every planned pass are compiled with g++ against
pass_ops.cuh (NQ_EMU) and executed on CPU threads (tests/jit_emu.py), then
compared with the oracle.  Covers what the GPU tests cover for the code
generator -- register layouts and relayouts, relabelled stores, 256-bit pair
accesses, pending register permutations (px on and off), phase accumulators,
pivot-normalised matrices -- without a GPU, so generator changes are caught
by the CPU suite."""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

import jit_emu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _perm_circuit(prng, n):
    kinds = [("cx", 2, 0), ("cx", 2, 0), ("ccx", 3, 0), ("swap", 2, 0), ("x", 1, 0), ("y", 1, 0), ("ry", 1, 1),
             ("u3", 1, 3), ("h", 1, 0), ("t", 1, 0), ("rz", 1, 1), ("cz", 2, 0), ("s", 1, 0)]
    circ = []
    for _ in range(300):
        k, ar, npar = kinds[int(prng.integers(len(kinds)))]
        qs = [int(q) for q in prng.choice(n, size=ar, replace=False)]
        circ.append((k, qs, [float(v) for v in prng.uniform(-3, 3, size=npar)]))
    for _ in range(2):
        circ += [("cx", [i, i + 1], []) for i in range(n - 1)] + [("ry", [q], [0.1 * q + 0.3]) for q in range(n)]
    return circ


@pytest.mark.parametrize("n,tile,seed", [(12, 8, 1), (13, 9, 5), (14, 11, 7)])
def test_generated_kernels_random_circuits(port, n, tile, seed):
    ops = port.random_circuit(seed, n, 250)
    got = jit_emu.run(n, ops, tile)
    assert np.max(np.abs(got - port.sv_run(n, ops))) <= 1e-12


@pytest.mark.parametrize("n,tile,seed", [(12, 8, 11), (13, 10, 12)])
def test_generated_kernels_permutation_heavy(port, n, tile, seed):
    circ = _perm_circuit(np.random.default_rng(seed), n)
    got = jit_emu.run(n, circ, tile)
    assert np.max(np.abs(got - port.sv_run(n, circ))) <= 1e-12


def test_generated_kernels_without_pending_permutations():
    # NQ_JIT_PX is read once per process by the generator: run in a child
    code = textwrap.dedent(f"""
        import sys
        sys.path[:0] = [{ROOT!r}, {os.path.join(ROOT, 'oracle')!r}, {os.path.join(ROOT, 'tests')!r}]
        import numpy as np
        from oracle import Port
        import jit_emu
        from test_jit_emu_cpu import _perm_circuit
        port = Port()
        worst = 0.0
        for n, tile, seed in [(12, 8, 11), (13, 9, 3)]:
            circ = _perm_circuit(np.random.default_rng(seed), n)
            worst = max(worst, float(np.max(np.abs(jit_emu.run(n, circ, tile) - port.sv_run(n, circ)))))
        print("WORST", worst)
        assert worst <= 1e-12, worst
    """)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, NQ_JIT_PX="0"), capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])


@pytest.mark.parametrize("n,tile", [(12, 8), (14, 10)])
def test_generated_kernels_qft_and_vqe_shapes(port, n, tile):
    """The two secondary benchmark shapes (bench.py): QFT (pure-phase
    controlled tables, per-thread phase accumulation, pivot-normalised
    rotations folding a pending phase) and the VQE ansatz (RY/RZ layers and
    CX ladders, relayout-heavy)."""
    from paper_2401_06861_b200 import workloads

    for circ in (workloads.qft(n), workloads.vqe_ansatz(n, 3, workloads.vqe_initial_params(n, 3))):
        got = jit_emu.run(n, circ, tile)
        assert np.max(np.abs(got - port.sv_run(n, circ))) <= 1e-12


@pytest.mark.parametrize("sanitizer", ["address", "thread"])
def test_generated_kernels_under_sanitizers(sanitizer):
    """The memcheck / racecheck substitute (compute-sanitizer is not available
    on the GPU pool): the generated pass kernels are emulated with g++'s
    AddressSanitizer (shared memory allocated at exactly the launch's size, the
    state and matrix pool as exact heap blocks: any out-of-bounds access
    aborts) and ThreadSanitizer (the CTA's threads are real threads
    synchronised by __syncthreads barriers: a missing barrier around a
    relayout is a reported data race)."""
    import shutil

    rt = subprocess.run(["g++", f"-print-file-name=lib{'a' if sanitizer == 'address' else 't'}san.so"],
                        capture_output=True, text=True).stdout.strip()
    if not rt or not os.path.isabs(rt) or shutil.which("g++") is None:
        pytest.skip("sanitizer runtime not available")
    code = textwrap.dedent(f"""
        import sys
        sys.path[:0] = [{ROOT!r}, {os.path.join(ROOT, 'oracle')!r}, {os.path.join(ROOT, 'tests')!r}]
        import numpy as np
        from oracle import Port
        import jit_emu
        from test_jit_emu_cpu import _perm_circuit
        from paper_2401_06861_b200 import workloads
        port = Port()
        worst = 0.0
        cases = [(11, 8, port.random_circuit(3, 11, 120)), (11, 9, _perm_circuit(np.random.default_rng(4), 11)),
                 (10, 8, workloads.qft(10))]
        for n, tile, circ in cases:
            worst = max(worst, float(np.max(np.abs(jit_emu.run(n, circ, tile) - port.sv_run(n, circ)))))
        assert worst <= 1e-12, worst
        print("EMU_OK", worst)
    """)
    env = dict(os.environ, NQ_EMU_SANITIZE=sanitizer, LD_PRELOAD=rt, PYTHONMALLOC="malloc",
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=1", TSAN_OPTIONS="halt_on_error=1:report_signal_unsafe=0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "EMU_OK" in out, out[-6000:]
    assert "ERROR: AddressSanitizer" not in out and "WARNING: ThreadSanitizer" not in out, out[-6000:]


@pytest.mark.parametrize("n,tile,seed", [(12, 8, 21), (13, 10, 22)])
def test_fused_z_epilogue(port, n, tile, seed):
    """The fused Z-term epilogue of a flush's last pass (sign = per-thread
    parity of the store index x compile-time register parity, with pending
    permutations): its sums equal sum_o |a_o|^2 (-1)^popcount(o & M) over the
    stored physical state, and the state itself is unchanged."""
    for circ in (port.random_circuit(seed, n, 200), _perm_circuit(np.random.default_rng(seed), n)):
        got, sums, phys_state = jit_emu.run(n, circ, tile, zterms=True)
        assert np.max(np.abs(got - port.sv_run(n, circ))) <= 1e-12
        p = np.abs(phys_state) ** 2
        o = np.arange(1 << n, dtype=np.int64)
        for k, mask in enumerate([1, 1 << (n - 1), 3]):
            sign = 1 - 2 * (np.array([bin(x).count("1") for x in (o & mask)]) & 1)
            assert abs(sums[k] - float(np.sum(p * sign))) <= 1e-12, (k, sums[k], float(np.sum(p * sign)))
