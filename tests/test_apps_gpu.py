"""Application entry points of the reference's Python surface on the B200
(csrc/apps.cpp): tfim_sweep, tfim_ground_energy, run_vqe.

Checked against the reference build (oracle/_ref: its own magnetization
sweep rows), the frozen values of proj/tests/test_tfim.cpp, a dense numpy
restatement of the exact column, and VQE traces driven by the oracle's
energies through the same Nelder-Mead."""
import os

import numpy as np
import pytest

from paper_2401_06861_b200 import naqs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CAL = os.path.join(ROOT, "tests", "golden", "example_5q.json")
PAULI = {"I": np.eye(2), "X": np.array([[0, 1], [1, 0]]), "Y": np.array([[0, -1j], [1j, 0]]),
         "Z": np.diag([1.0, -1.0])}


def tfim_terms(n, J=1.0, h=1.0, periodic=False):
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


def dense(terms, n):
    H = np.zeros((1 << n, 1 << n), dtype=complex)
    for letters, c in terms:
        m = np.array([[1.0]])
        for q in range(n):  # letters[q] acts on qubit q: rightmost Kronecker factor is qubit 0
            m = np.kron(PAULI[letters[q]], m)
        H += c * m
    return H


def exact_column(n, ts):
    w, V = np.linalg.eigh(dense(tfim_terms(n), n))
    psi0 = np.zeros(1 << n, dtype=complex)
    psi0[0] = 1
    out = []
    for t in ts:
        psi = V @ (np.exp(-1j * w * t) * (V.conj().T @ psi0))
        p = np.abs(psi) ** 2
        out.append(np.mean([np.sum(np.where((np.arange(1 << n) >> q) & 1, -p, p)) for q in range(n)]))
    return np.array(out)


def test_ground_energy_frozen_and_dense():
    assert naqs.tfim_ground_energy(4) == pytest.approx(-4.7587704831436355, rel=1e-12)  # test_tfim.cpp:15
    for n, b in [(3, "periodic"), (6, "open"), (5, "periodic")]:
        want = np.linalg.eigvalsh(dense(tfim_terms(n, 0.7, 1.3, b == "periodic"), n))[0]
        assert abs(naqs.tfim_ground_energy(n, 0.7, 1.3, b) - want) < 1e-10
    with pytest.raises(naqs.NaqsError, match="boundary must be"):
        naqs.tfim_ground_energy(3, boundary="ring")


def test_sweep_matches_reference_rows(ref):
    cal = open(CAL).read()
    rows = naqs.tfim_sweep(4, noise=naqs.load_calibration(cal))
    t, ideal, noisy, _ = ref.tfim_sweep(cal, 4)
    assert len(rows) == len(t) == 31
    got = np.array([(r[0], r[1], r[2], r[3]) for r in rows])
    assert np.array_equal(got[:, 0], t)  # accumulated t (0.30000000000000004, ...)
    np.testing.assert_allclose(got[:, 2], ideal, atol=1e-10, rtol=0)
    np.testing.assert_allclose(got[:, 3], noisy, atol=1e-10, rtol=0)
    np.testing.assert_allclose(got[:, 1], exact_column(4, t), atol=1e-10, rtol=0)


def test_sweep_without_noise_and_frozen_exact_values():
    rows = naqs.tfim_sweep(4, t_max=2.0, dt=0.5)
    assert [r[3] for r in rows] == [None] * 5
    ex = {r[0]: r[1] for r in rows}
    # proj/tests/test_tfim.cpp:16-18
    assert ex[0.5] == pytest.approx(0.6168386101703245, abs=1e-10)
    assert ex[1.0] == pytest.approx(0.13507747985560886, abs=1e-10)
    assert ex[2.0] == pytest.approx(0.019004665262770136, abs=1e-10)


def test_sweep_with_shots_samples_each_row_with_derived_seeds(port):
    cal = open(CAL).read()
    model = naqs.load_calibration(cal)
    rows = naqs.tfim_sweep(3, t_max=0.4, dt=0.2, noise=model, shots=3000, seed=11)
    from paper_2401_06861_b200 import workloads

    for r, row in enumerate(rows):
        c = naqs.Circuit(3)
        for name, qs, ps in workloads.tfim_trotter(3, row[0]):
            c.add(name, qs, ps)
        dist = np.array(naqs.noisy_distribution(c, model))
        counts = port.sample_distribution(dist, 3000, port.derive_seed(11, r)).astype(float) / 3000
        want = np.mean([np.sum(np.where((np.arange(8) >> q) & 1, -counts, counts)) for q in range(3)])
        assert row[3] == pytest.approx(want, abs=1e-12)


def ansatz_ops(n, layers, x):
    ops, k = [], 0
    for q in range(n):
        ops.append(("ry", [q], [x[k]]))
        k += 1
    for _ in range(layers):
        for i in range(n - 1):
            ops.append(("cx", [i, i + 1], []))
        for q in range(n):
            ops.append(("ry", [q], [x[k]]))
            k += 1
    return ops


def test_run_vqe_follows_the_oracle_energies(port):
    n, layers = 4, 2
    terms = tfim_terms(n)

    def energy(x):
        a = port.sv_run(n, ansatz_ops(n, layers, x))
        return sum(port.expectation(a, L, c) for L, c in terms)

    x0 = port.rng_double(1, n * (layers + 1)) * 0.2 - 0.1  # Rng(1).uniform(-0.1, 0.1)
    want = naqs.minimize(energy, list(x0), max_evals=80, initial_step=2.0)
    got = naqs.run_vqe(n, layers=layers, max_evals=80)
    np.testing.assert_allclose(got.trace, want.trace, atol=1e-10, rtol=0)
    assert got.iterations == 80 and not got.converged


def test_noisy_vqe_energy_uses_the_density_matrix(port):
    from oracle import NoiseSpec

    n, layers = 3, 1
    spec = NoiseSpec(n)
    model = naqs.load_calibration(spec.calibration_json())
    terms = tfim_terms(n)

    def energy(x):
        rho = port.dm_run_noisy(n, ansatz_ops(n, layers, x), spec)
        return sum(port.dm_expectation(rho, L, c) for L, c in terms)

    x0 = port.rng_double(1, n * (layers + 1)) * 0.2 - 0.1
    want = naqs.minimize(energy, list(x0), max_evals=12, initial_step=2.0)
    got = naqs.run_vqe(n, layers=layers, max_evals=12, noise=model)
    np.testing.assert_allclose(got.trace, want.trace, atol=1e-10, rtol=0)
