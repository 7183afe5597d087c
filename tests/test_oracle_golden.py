"""Pin the oracle before trusting it (CPU only).

1. The C restatement reproduces the reference's own golden vectors and
   known-answer tests, cited file:line.
2. In the build container it also matches the reference compiled from its
   own sources (oracle/_ref) bit for bit on seeded random circuits.
3. The reference's own unit-test suites pass against that build
   (oracle/_ref/ref_unit_tests), which validates the Eigen-API subset used to
   compile it.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import NoiseSpec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def test_rng_golden_vectors(port):
    # proj/tests/test_statevector.cpp:234-246
    a = port.rng_u64(1, 5)
    assert [int(x) for x in a[:4]] == [0xCFC5D07F6F03C29B, 0xBF424132963FE08D, 0x19A37D5757AAF520, 0xBF08119F05CD56D6]
    assert port.rng_double(1, 5)[4] == pytest.approx(0.18467857211916938, rel=1e-16)
    b = port.rng_u64(20240607, 2)
    assert [int(x) for x in b] == [0xD4D92CCEEB95E8DC, 0x44862A3B34B27EE0]


def test_bell_and_little_endian(port):
    # proj/tests/test_statevector.cpp:38-45, 64-73
    a = port.sv_run(2, [("x", [0]), ("cx", [0, 1])])
    assert abs(a[3] - 1) <= 1e-15 and abs(a[1]) <= 1e-15
    b = port.sv_run(2, [("h", [0]), ("cx", [0, 1])])
    r = 1 / np.sqrt(2)
    np.testing.assert_allclose(b, [r, 0, 0, r], atol=1e-15)
    assert port.expectation(b, "ZZ") == pytest.approx(1.0)
    assert port.expectation(b, "XX") == pytest.approx(1.0)
    assert port.expectation(b, "YY") == pytest.approx(-1.0)
    assert abs(port.expectation(b, "ZI")) < 1e-15


def test_every_gate_against_independent_numpy_model(port):
    # proj/tests/python/test_reference.py:13-131: the same 20-gate sequence and
    # the same independent textbook model, restated here
    ops = [("h", [0]), ("x", [1]), ("y", [2]), ("z", [0]), ("s", [1]), ("sdg", [2]), ("t", [0]), ("tdg", [1]),
           ("id", [2]), ("rx", [0], [0.3]), ("ry", [1], [-0.7]), ("rz", [2], [1.1]), ("u1", [0], [0.4]),
           ("u2", [1], [0.2, -0.5]), ("u3", [2], [1.2, 0.3, -0.8]), ("cx", [0, 1]), ("cz", [1, 2]),
           ("swap", [0, 2]), ("ccx", [0, 1, 2]), ("cx", [2, 0])]
    got = port.sv_run(3, ops)
    want = np.load(os.path.join(GOLD, "every_gate_numpy_model.npy"))
    assert np.max(np.abs(got - want)) < 1e-12


def test_depolarizing_known_answers(port):
    # proj/tests/test_densitymatrix.cpp:90-98 and test_noise.cpp:297-306
    for p, z in [(0.15, 0.8), (0.3, 0.6)]:
        rho = port.dm_new(1).reshape(2, 2)
        rho = port.dm_apply_channel(rho, [0], port.depolarizing(p, 1))
        assert port.dm_expectation(rho, "Z") == pytest.approx(z, abs=1e-12)
    rho = port.dm_run(1, [("x", [0])])
    rho = port.dm_apply_channel(rho, [0], port.depolarizing(0.09, 1))
    assert port.dm_expectation(rho, "Z") == pytest.approx(-(1 - 4 * 0.09 / 3), abs=1e-12)
    # maximally mixed at p = 3/4 (test_densitymatrix.cpp:183-195)
    rho = port.dm_apply_channel(port.dm_new(1).reshape(2, 2), [0], port.depolarizing(0.75, 1))
    np.testing.assert_allclose(port.dm_probabilities(rho), [0.5, 0.5], atol=1e-12)


def test_thermal_decay_law(port):
    # proj/tests/test_noise.cpp:42-60: coherence decays as exp(-d/T2)
    t1, t2, ns = 50.0, 30.0, 400.0
    plus = np.array([[0.5, 0.5], [0.5, 0.5]], dtype=complex)
    out = port.dm_apply_channel(plus.copy(), [0], port.thermal_relaxation(t1, t2, ns))
    d = ns / 1000
    assert abs(out[0, 1]) == pytest.approx(0.5 * np.exp(-d / t2), abs=1e-12)
    one = np.array([[0, 0], [0, 1]], dtype=complex)
    out = port.dm_apply_channel(one, [0], port.thermal_relaxation(t1, t2, ns))
    assert out[1, 1].real == pytest.approx(np.exp(-d / t1), abs=1e-12)
    assert len(port.thermal_relaxation(t1, t2, 0.0)) == 1


def test_readout_known_answers(port):
    # proj/tests/test_noise.cpp:84-95 and 97-132
    r = port.readout_apply_dist([1.0, 0.0], [0.05], [0.02])
    np.testing.assert_allclose(r, [0.98, 0.02], atol=1e-15)
    p = 0.07
    dist = np.zeros(4)
    dist[0] = 1
    out = port.readout_apply_dist(dist, [p, p], [p, p])
    z0 = out[0] - out[1] + out[2] - out[3]
    assert z0 == pytest.approx(1 - 2 * p, abs=1e-12)


def test_tfim_e0_golden(port):
    # proj/tests/test_tfim.cpp:15-18: E0 of the n=4 open chain (J = h = 1) is
    # -4.7587704831436355.  The ground state from an independent numpy
    # Hamiltonian must give exactly that energy through the oracle's
    # expectation kernel (statevector.cpp:241-277), term by term.
    n = 4
    terms = [("ZZII", -1.0), ("IZZI", -1.0), ("IIZZ", -1.0), ("XIII", -1.0), ("IXII", -1.0), ("IIXI", -1.0),
             ("IIIX", -1.0)]
    P = {"I": np.eye(2), "X": np.array([[0, 1], [1, 0]]), "Y": np.array([[0, -1j], [1j, 0]]),
         "Z": np.diag([1.0, -1.0])}
    H = np.zeros((16, 16), dtype=complex)
    for L, c in terms:
        m = np.array([[c]], dtype=complex)
        for ch in L:  # letters[0] is the rightmost Kronecker factor
            m = np.kron(P[ch], m)
        H += m
    w, v = np.linalg.eigh(H)
    assert w[0] == pytest.approx(-4.7587704831436355, abs=1e-12)
    psi = np.ascontiguousarray(v[:, 0])
    e = sum(port.expectation(psi, L, c) for L, c in terms)
    assert e == pytest.approx(-4.7587704831436355, abs=1e-12)


def test_random_circuit_generator_matches_reference(port, ref):
    for seed, n, d, ma in [(2024, 30, 200, 3), (17, 3, 12, 3), (4040 + 34, 34, 200, 3), (97, 5, 30, 2)]:
        assert port.random_circuit(seed, n, d, ma).tobytes() == ref.random_circuit(seed, n, d, ma).tobytes()


@pytest.mark.parametrize("seed", range(6))
def test_port_is_bit_exact_with_reference_build(port, ref, seed):
    n = 3 + seed
    ops = port.random_circuit(900 + seed, n, 80)
    assert np.array_equal(port.sv_run(n, ops), ref.sv_run(n, ops))
    letters = "".join("IXYZ"[(seed + i) % 4] for i in range(n))
    assert port.expectation(port.sv_run(n, ops), letters, 0.7) == ref.sv_expectations(n, ops, [(letters, 0.7)])[0]
    m = 2 + seed % 4
    c = port.random_circuit(700 + seed, m, 40, 2)
    noise = NoiseSpec(m, e1=0.003 * (seed + 1), e2=0.02)
    assert np.array_equal(port.dm_run_noisy(m, c, noise), ref.dm_run_noisy(m, c, noise))
    dist = np.abs(port.sv_run(n, ops)) ** 2
    assert np.array_equal(port.sample_distribution(dist, 5000, seed), ref.sample_distribution(dist, 5000, seed))


def test_reference_unit_tests_pass_on_reference_build(ref):
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests")
    if not os.path.exists(exe):
        pytest.skip("reference unit-test binary not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_golden_fixture_manifest():
    with open(os.path.join(GOLD, "MANIFEST.json")) as f:
        man = json.load(f)
    for name in man["files"]:
        assert os.path.exists(os.path.join(GOLD, name)), name
