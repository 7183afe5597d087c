"""Run-time specialised pass kernels (jit.cpp) against the oracle.

NQ_JIT is read once per process, so each case runs in a subprocess with
NQ_JIT=sync (every pass of tile size >= 8 compiled and launched as a
specialised kernel) and compares with the oracle there.
"""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent(
    """
    import sys
    sys.path[:0] = [{root!r}, {oracle!r}]
    import numpy as np
    from oracle import Port, NoiseSpec, ops_to_list
    from paper_2401_06861_b200 import abi, naqs
    port = Port()
    worst = 0.0
    for n, tile, seed in [(12, 8, 1), (14, 10, 2), (16, 12, 3), (18, 12, 4), (17, 9, 5), (20, 13, 6), (22, 11, 7)]:
        ops = port.random_circuit(seed, n, 250)
        sv = abi.SV(n, tile_qubits=tile)
        sv.apply(ops)
        got = sv.amplitudes()
        worst = max(worst, float(np.max(np.abs(got - port.sv_run(n, ops)))))
        # a second run of the same structure reuses the compiled kernels
        sv.reset()
        sv.apply(ops)
        assert np.array_equal(sv.amplitudes(), got)
    # permutation-heavy circuits: X-type gates whose controls sit on thread,
    # tile or global bits are recorded in the pending register permutation
    # (jit.cpp px) and must come out right through every later op kind
    prng = np.random.default_rng(99)
    kinds = [("cx", 2, 0), ("cx", 2, 0), ("ccx", 3, 0), ("swap", 2, 0), ("x", 1, 0), ("y", 1, 0), ("ry", 1, 1),
             ("u3", 1, 3), ("h", 1, 0), ("t", 1, 0), ("rz", 1, 1), ("cz", 2, 0), ("s", 1, 0)]
    for n, tile, seed in [(12, 8, 11), (15, 10, 12), (18, 11, 13), (21, 12, 14)]:
        circ = []
        for _ in range(300):
            k, ar, npar = kinds[int(prng.integers(len(kinds)))]
            qs = [int(q) for q in prng.choice(n, size=ar, replace=False)]
            circ.append((k, qs, [float(v) for v in prng.uniform(-3, 3, size=npar)]))
        for layers in range(2):  # a CX ladder (VQE ansatz shape)
            circ += [("cx", [i, i + 1], []) for i in range(n - 1)] + [("ry", [q], [0.1 * q + 0.3]) for q in range(n)]
        sv = abi.SV(n, tile_qubits=tile)
        sv.apply(abi.make_ops(circ))
        worst = max(worst, float(np.max(np.abs(sv.amplitudes() - port.sv_run(n, circ)))))
    # density matrix with noise (Liouville superoperators, depolarizing maps);
    # n >= 6 runs the Hermitian (mirror) passes on the interleaved layout
    for n in (5, 6, 8, 9):
        c = port.random_circuit(100 + n, n, 60, 2)
        circ = naqs.Circuit(n)
        for k, q, p in ops_to_list(c):
            circ.add(k, q, p)
        noise = NoiseSpec(n, e1=0.01, e2=0.05)
        rho = naqs.run_density(circ, naqs.load_calibration(noise.calibration_json()))
        worst = max(worst, float(np.max(np.abs(rho - port.dm_run_noisy(n, c, noise)))))
    # expectation batches: specialised register-layout kernels (tile 12)
    from paper_2401_06861_b200 import workloads
    rng = np.random.default_rng(7)
    for n, seed in [(13, 11), (16, 12), (19, 13)]:
        ops = port.random_circuit(seed, n, 120)
        sv = abi.SV(n)
        sv.apply(ops)
        amps = sv.amplitudes()
        terms = list(workloads.tfim_hamiltonian(n, periodic=True))
        for _ in range(40):
            w = int(rng.integers(1, 6))
            L = ["I"] * n
            for q in rng.choice(n, size=w, replace=False):
                L[int(q)] = "XYZ"[int(rng.integers(0, 3))]
            terms.append(("".join(L), float(rng.normal())))
        got = sv.expectations(terms)
        for (letters, coeff), g in zip(terms, got):
            ref = port.expectation(amps, letters, coeff)
            worst = max(worst, abs(g - ref))
        assert np.array_equal(sv.expectations(terms), got)  # deterministic
    st = abi.jit_stats()
    assert st["launches"] > 0 and st["failed"] == 0, st
    print("WORST", worst, st)
    assert worst <= 1e-10, worst
    """
)


@pytest.mark.parametrize("px", ["1", "0"])
def test_specialised_kernels_match_oracle(px):
    env = dict(os.environ, NQ_JIT="sync", NQ_JIT_PX=px)
    code = SCRIPT.format(root=ROOT, oracle=os.path.join(ROOT, "oracle"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "WORST" in r.stdout


FUSED_Z = textwrap.dedent(
    """
    import sys
    sys.path[:0] = [{root!r}, {oracle!r}]
    import numpy as np
    from oracle import Port
    from paper_2401_06861_b200 import abi
    port = Port()
    worst = 0.0
    for n, seed in [(19, 3), (20, 8), (22, 13)]:
        ops = port.random_circuit(seed, n, 150)
        terms = [("Z" + "I" * (n - 1), 1.0), ("I" * (n - 1) + "Z", -0.5),
                 ("ZZ" + "I" * (n - 3) + "Z", 0.25), ("I" * 5 + "Z" + "I" * (n - 6), 2.0)]
        sv = abi.SV(n)
        for rep in range(3):  # the repeated circuit: carried layout, cached plan
            abi.profile_begin(0, per_pass_events=False)
            sv.apply(ops)
            fused = sv.expectations(terms)  # flush + terms in its last pass
            prof = abi.profile_end(0)
            passes = sv.stats()["launches"]
            assert prof["kernel_launches"] == passes + 1, (prof, passes)  # passes + the final fixed-order sum
            again = sv.expectations(terms)  # nothing queued: the standalone reduction
            amps = sv.amplitudes()
            for (letters, coeff), g, h in zip(terms, fused, again):
                ref = port.expectation(amps, letters, coeff)
                worst = max(worst, abs(g - ref), abs(h - ref))
        sv.close()
    print("WORST", worst)
    assert worst <= 1e-10, worst
    """
)


def test_z_terms_fused_into_the_last_pass():
    """A flush whose result is read as Z-type terms computes them in the
    epilogue of its last pass (one state read saved; the e2e benchmark's
    <Z0>): same values as the standalone reduction and the oracle, and no
    separate reduction kernel (launches = passes + 1 fixed-order final sum)."""
    env = dict(os.environ, NQ_JIT="sync")
    code = FUSED_Z.format(root=ROOT, oracle=os.path.join(ROOT, "oracle"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "WORST" in r.stdout
