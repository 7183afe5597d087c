"""State-vector parity on the GPU through the C ABI.

The checker is the C restatement (oracle/naqs_oracle.c), itself pinned
bit-for-bit to the reference build (test_oracle_golden.py).  Tolerance: 1e-10
absolute on amplitudes and expectations (BASELINE.json north star); index and
bit-ordering logic must be exact (sampling counts, permutations).
"""
import numpy as np
import pytest

from paper_2401_06861_b200 import abi

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 11, 13, 16])
@pytest.mark.parametrize("fuse", [True, False])
def test_random_circuits_match_oracle(port, n, fuse):
    for seed in range(3):
        ops = port.random_circuit(1000 * n + seed, n, 120)
        sv = abi.SV(n, fuse=fuse)
        sv.apply(ops)
        np.testing.assert_allclose(sv.amplitudes(), port.sv_run(n, ops), atol=TOL, rtol=0)


@pytest.mark.parametrize("tile", [4, 5, 6, 8, 10, 12, 13])
def test_tile_sizes_exercise_high_qubit_gather(port, tile):
    # n larger than the tile forces multi-tile passes with high tile bits
    n = 15
    ops = port.random_circuit(77 + tile, n, 300)
    sv = abi.SV(n, tile_qubits=tile)
    sv.apply(ops)
    np.testing.assert_allclose(sv.amplitudes(), port.sv_run(n, ops), atol=TOL, rtol=0)
    st = sv.stats()
    assert st["source_ops"] == 300 and st["passes"] >= 1


def test_every_gate_kind_on_every_position(port):
    n = 6
    kinds = [("x", 1, 0), ("y", 1, 0), ("z", 1, 0), ("h", 1, 0), ("s", 1, 0), ("sdg", 1, 0), ("t", 1, 0),
             ("tdg", 1, 0), ("id", 1, 0), ("rx", 1, 1), ("ry", 1, 1), ("rz", 1, 1), ("u1", 1, 1), ("u2", 1, 2),
             ("u3", 1, 3), ("cx", 2, 0), ("cz", 2, 0), ("swap", 2, 0), ("ccx", 3, 0)]
    rng = np.random.default_rng(5)
    prefix = [("h", [q]) for q in range(n)] + [("ry", [q], [0.3 * q + 0.1]) for q in range(n)]
    for name, ar, npar in kinds:
        for trial in range(4):
            qs = list(rng.choice(n, size=ar, replace=False))
            ops = prefix + [(name, [int(q) for q in qs], list(rng.uniform(-3, 3, npar)))]
            for tile in (0, 4):
                sv = abi.SV(n, tile_qubits=tile)
                sv.apply(ops)
                np.testing.assert_allclose(sv.amplitudes(), port.sv_run(n, ops), atol=1e-12, rtol=0)


def test_permutations_are_exact(port):
    # X / CX / SWAP / CCX move amplitudes without arithmetic: bit-exact
    n = 14
    rng = np.random.default_rng(1)
    amps = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    ops = []
    for _ in range(200):
        k = rng.integers(4)
        qs = [int(q) for q in rng.choice(n, size=3, replace=False)]
        ops.append([("x", qs[:1]), ("cx", qs[:2]), ("swap", qs[:2]), ("ccx", qs)][k])
    sv = abi.SV(n)
    sv.set_amplitudes(amps)
    sv.apply(ops)
    want = port.sv_apply(amps.copy(), ops)
    assert np.array_equal(sv.amplitudes(), want)


def test_norm_and_expectations(port):
    n = 12
    ops = port.random_circuit(31, n, 150)
    sv = abi.SV(n)
    sv.apply(ops)
    want = port.sv_run(n, ops)
    assert abs(sv.norm_sq() - port.norm_sq(want)) <= 1e-12
    rng = np.random.default_rng(3)
    terms = []
    for _ in range(40):
        letters = "".join(rng.choice(list("IXYZ"), size=n))
        terms.append((letters, float(rng.uniform(-2, 2))))
    terms.append(("I" * n, 1.5))
    got = sv.expectations(terms)
    ref = [port.expectation(want, L, c) for L, c in terms]
    np.testing.assert_allclose(got, ref, atol=TOL, rtol=0)


def test_probabilities(port):
    n = 13
    ops = port.random_circuit(8, n, 100)
    sv = abi.SV(n)
    sv.apply(ops)
    np.testing.assert_allclose(sv.probabilities(), np.abs(port.sv_run(n, ops)) ** 2, atol=1e-14, rtol=0)


@pytest.mark.parametrize("n,shots", [(3, 1000), (10, 20000), (14, 5000)])
def test_sampling_counts_match_reference_sweep(port, n, shots):
    ops = port.random_circuit(55 + n, n, 80)
    sv = abi.SV(n)
    sv.apply(ops)
    seed = 99
    u = np.sort(port.rng_double(seed, shots))
    idx, cnt = sv.sample_sorted(u)
    dense = np.zeros(1 << n, dtype=np.uint64)
    dense[idx.astype(np.int64)] = cnt
    want = port.sample_distribution(np.abs(port.sv_run(n, ops)) ** 2, shots, seed)
    assert int(dense.sum()) == shots
    assert np.array_equal(dense, want)


def test_deterministic_state_sampling():
    sv = abi.SV(4)
    idx, cnt = sv.sample_sorted(np.sort(np.random.default_rng(0).random(100)))
    assert list(idx) == [0] and list(cnt) == [100]


def test_kraus_weights_and_matrix(port):
    n = 7
    ops = port.random_circuit(4, n, 60)
    sv = abi.SV(n)
    sv.apply(ops)
    want = port.sv_run(n, ops)
    kr = port.depolarizing(0.2, 2)
    w = sv.kraus_weights([5, 1], kr)
    # ||K psi||^2 on the oracle
    ref = []
    for K in kr:
        a = want.copy()
        port.sv_apply_matrix(a, [5, 1], K)
        ref.append(np.sum(np.abs(a) ** 2))
    np.testing.assert_allclose(w, ref, atol=1e-12, rtol=0)
    assert abs(w.sum() - 1) < 1e-12
    sv.apply_matrix([5, 1], kr[3] / np.sqrt(w[3]))
    a = want.copy()
    port.sv_apply_matrix(a, [5, 1], kr[3])
    np.testing.assert_allclose(sv.amplitudes(), a / np.sqrt(ref[3]), atol=TOL, rtol=0)


def test_clone_reset_and_contract_errors():
    sv = abi.SV(3)
    sv.apply([("h", [0]), ("cx", [0, 2])])
    c = sv.clone()
    sv.reset()
    assert np.allclose(sv.amplitudes(), [1, 0, 0, 0, 0, 0, 0, 0])
    r = 2 ** -0.5
    assert np.allclose(c.amplitudes(), [r, 0, 0, 0, 0, r, 0, 0])
    with pytest.raises(abi.ContractError, match="out of range"):
        sv.apply([("x", [3])])
    with pytest.raises(abi.ContractError, match="MEASURE"):
        sv.apply([("measure", [0])])
    with pytest.raises(abi.ContractError):
        abi.SV(31)
    with pytest.raises(abi.ContractError):
        abi.SV(0)


def test_bit_identical_reruns(port):
    n = 16
    ops = port.random_circuit(9, n, 200)
    a = abi.SV(n).apply(ops)
    b = abi.SV(n).apply(ops)
    assert np.array_equal(a.amplitudes(), b.amplitudes())
    t = [("ZIZIZIZIZIZIZIZI", 1.0), ("XXYYIIIIIIIIIIII", -0.5)]
    assert np.array_equal(a.expectations(t), b.expectations(t))
    assert a.norm_sq() == b.norm_sq()


def test_large_state_beyond_reference_guard(port):
    # explicit large-state entry point (max_qubits): a GHZ chain on 28 qubits
    n = 28
    sv = abi.SV(n, max_qubits=34)
    sv.apply([("h", [0])] + [("cx", [q, q + 1]) for q in range(n - 1)])
    amps = sv.amplitudes(0, 1)
    last = sv.amplitudes((1 << n) - 1, 1)
    assert abs(amps[0] - 2 ** -0.5) < 1e-14 and abs(last[0] - 2 ** -0.5) < 1e-14
    assert abs(sv.norm_sq() - 1) < 1e-12
    e = sv.expectations([("Z" * n, 1.0), ("X" * n, 1.0), ("Z" + "I" * (n - 1), 1.0)])
    np.testing.assert_allclose(e, [1.0, 1.0, 0.0], atol=1e-12)


def test_device_view_zero_copy():
    """f4: the amplitudes in HBM through __cuda_array_interface__ (torch),
    no host copy, equal to nq_sv_get_amplitudes."""
    import torch

    n = 12
    sv = abi.SV(n)
    sv.apply(abi.make_ops([("h", [q], []) for q in range(n)] + [("rz", [3], [0.4]), ("cx", [3, 7], [])]))
    view = sv.device_view()
    t = torch.as_tensor(view, device="cuda")
    assert t.dtype == torch.complex128 and t.numel() == 1 << n
    assert t.data_ptr() == view.ptr
    assert np.array_equal(t.cpu().numpy(), sv.amplitudes())
