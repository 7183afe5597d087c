"""Parity at the benchmarked scale ("parity vs the oracle is
checked before a timing counts").

Every configuration bench.py times is compared here, at its benchmarked size,
with the reference engine compiled from its own sources (oracle/_ref):

* C2 random circuit, n = 30, depth 200, Rng(2024): norm, <Z_q> on 8 qubits,
  a Pauli string with X/Y/Z, and 4096 amplitudes (64 windows of 64);
* C2 QFT-30: 4096 amplitudes against the closed form of the QFT of the prep
  product state (oracle.qft_closed_form, pinned to oracle/_ref by
  tests/test_scale_parity_cpu.py; the reference engine needs minutes for the
  2,220 ops), and the full QFT-24 state against oracle/_ref;
* C5 VQE-28: the exact energy over 55 Hamiltonian terms;
* C4 noisy TFIM density matrix at n = 12 (interleaved layout, Hermitian
  mirror passes, multi-tile: the n = 14 path): the full rho;
* sampling at n = 24 with 1e5 shots: exact counts.
Tolerance: 1e-10 absolute (north_star); counts bit-exact.
"""
import numpy as np
import pytest

from oracle import NoiseSpec, Port, list_to_ops, qft_closed_form
from paper_2401_06861_b200 import abi, workloads

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _windows(n, seed, windows=64, width=64):
    rng = np.random.default_rng(seed)
    starts = rng.integers(0, (1 << n) - width, size=windows)
    starts[0] = 0
    return [(int(s), width) for s in starts]


def _z_terms(n, qs):
    out = []
    for q in qs:
        L = ["I"] * n
        L[q] = "Z"
        out.append(("".join(L), 1.0))
    return out


def _host_gib():
    with open("/proc/meminfo") as f:
        for ln in f:
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) / (1 << 20)
    return 0.0


def test_random30_matches_reference(ref):
    n = 30
    if _host_gib() < 24:
        pytest.skip("host RAM too small for a 16 GiB reference state")
    ops_list = workloads.random_circuit(2024, n, 200)
    sv = abi.SV(n)
    sv.apply(abi.make_ops(ops_list)).flush()
    ref.set_threads(0)
    h = ref.sv_new(n)
    try:
        ref.sv_run_timed(h, list_to_ops(ops_list))
        terms = _z_terms(n, [0, 1, 7, 15, 25, 27, 28, 29]) + [("XX" + "I" * (n - 4) + "YZ", 0.5)]
        np.testing.assert_allclose(sv.expectations(terms), ref.sv_expectations_h(h, n, terms), atol=TOL, rtol=0)
        assert abs(sv.norm_sq() - ref.sv_norm_sq_h(h)) <= TOL
        for off, w in _windows(n, 0):
            np.testing.assert_allclose(sv.amplitudes(off, w), ref.sv_gather(h, np.arange(off, off + w)),
                                       atol=TOL, rtol=0)
    finally:
        ref.sv_free(h)
        sv.close()


def test_qft30_matches_closed_form():
    n = 30
    sv = abi.SV(n)
    sv.apply(abi.make_ops(workloads.qft(n))).flush()
    for off, w in _windows(n, 1):
        np.testing.assert_allclose(sv.amplitudes(off, w), qft_closed_form(n, np.arange(off, off + w)),
                                   atol=TOL, rtol=0)
    assert abs(sv.norm_sq() - 1.0) <= TOL
    sv.close()


def test_qft24_full_state_matches_reference(ref):
    n = 24
    ops = workloads.qft(n)
    sv = abi.SV(n)
    sv.apply(abi.make_ops(ops))
    got = sv.amplitudes()
    want = ref.sv_run(n, list_to_ops(ops))
    assert np.max(np.abs(got - want)) <= TOL
    sv.close()


def test_vqe28_energy_matches_reference(ref):
    n, layers = 28, 3
    ops = workloads.vqe_ansatz(n, layers, workloads.vqe_initial_params(n, layers))
    terms = workloads.tfim_hamiltonian(n)
    assert len(ops) == 193 and len(terms) == 55
    sv = abi.SV(n)
    sv.apply(abi.make_ops(ops))
    e = sv.expectations(terms)
    sv.close()
    h = ref.sv_new(n)
    try:
        ref.sv_run_timed(h, list_to_ops(ops))
        e_ref = ref.sv_expectations_h(h, n, terms)
    finally:
        ref.sv_free(h)
    np.testing.assert_allclose(e, e_ref, atol=TOL, rtol=0)
    assert abs(float(np.sum(e)) - float(np.sum(e_ref))) <= TOL


def test_noisy_tfim_dm12_full_rho_matches_reference(ref):
    from paper_2401_06861_b200 import naqs

    n = 12
    ops = list(workloads.tfim_trotter(n, 1.0, steps=10))
    spec = NoiseSpec(n)
    c = naqs.Circuit(n)
    for name, qs, ps in ops:
        c.add(name, qs, ps)
    rho = naqs.run_density(c, naqs.load_calibration(spec.calibration_json()))
    rho_ref = ref.dm_run_noisy(n, ops, spec)
    assert np.max(np.abs(rho - rho_ref)) <= TOL


def test_sampling_n24_exact_counts(ref):
    n, shots, seed = 24, 100_000, 4242
    ops = ref.random_circuit(2424, n, 120)
    sv = abi.SV(n)
    sv.apply(ops)
    u = np.sort(Port().rng_double(seed, shots))  # Rng(seed).next_double stream
    idx, cnt = sv.sample_sorted(u)
    got = np.zeros(1 << n, dtype=np.uint64)
    got[idx.astype(np.int64)] = cnt
    assert int(got.sum()) == shots
    # the reference samples its own state: equal counts
    want = ref.sv_sample(n, ops, shots, seed)
    assert np.array_equal(got, want)
    # and the device sweep over the reference's own distribution (|a|^2 as
    # std::norm: re*re + im*im, no fused multiply-add) is bit-exact by construction
    a = ref.sv_run(n, ops)
    dist = a.real * a.real + a.imag * a.imag
    i2, c2 = abi.sample_dist_sorted(dist, u)
    got2 = np.zeros(1 << n, dtype=np.uint64)
    got2[i2.astype(np.int64)] = c2
    assert np.array_equal(got2, ref.sample_distribution(dist, shots, seed))
    sv.close()
