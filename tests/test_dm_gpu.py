"""Density-matrix parity on the GPU.

Gates and channels run as Liouville-space superoperators on vec(rho) in the
fused pass kernel; the checker is the oracle's blockwise Kraus sum
(proj/src/densitymatrix.cpp:60-110).  Tolerance 1e-10 absolute.
"""
import numpy as np
import pytest

from oracle import NoiseSpec, ops_to_list
from paper_2401_06861_b200 import abi

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.mark.parametrize("n", [1, 2, 3, 5, 7])
def test_unitary_dm_matches_oracle(port, n):
    ops = port.random_circuit(300 + n, n, 60)
    d = abi.DM(n)
    d.apply(ops)
    np.testing.assert_allclose(d.rho(), port.dm_run(n, ops), atol=TOL, rtol=0)


@pytest.mark.parametrize("n", [2, 4, 6, 8])
@pytest.mark.parametrize("tile", [0, 6])
def test_noisy_schedule_matches_oracle(port, n, tile):
    ops = port.random_circuit(400 + n, n, 50, 2)
    noise = NoiseSpec(n, e1=0.01, e2=0.05)
    items = []
    for name, qubits, params in ops_to_list(ops):
        items.append(("gate", (name, qubits, params)))
        if name == "id" or True:
            k = len(qubits)
            items.append(("channel", qubits, port.depolarizing(noise.e1 if k == 1 else noise.e2, k)))
            dur = noise.d1 if k == 1 else noise.d2
            for q in qubits:
                items.append(("channel", [q], port.thermal_relaxation(60.0, 40.0, dur)))
    d = abi.DM(n, tile_qubits=tile)
    d.apply_schedule(items)
    np.testing.assert_allclose(d.rho(), port.dm_run_noisy(n, ops, noise), atol=TOL, rtol=0)


@pytest.mark.parametrize("kind", ["depol1", "depol2", "thermal", "damp"])
def test_single_channels(port, kind):
    n = 4
    ops = port.random_circuit(17, n, 30)
    rho0 = port.dm_run(n, ops)
    if kind == "depol1":
        qs, kr = [2], port.depolarizing(0.3, 1)
    elif kind == "depol2":
        qs, kr = [3, 1], port.depolarizing(0.4, 2)
    elif kind == "thermal":
        qs, kr = [0], port.thermal_relaxation(50.0, 30.0, 250.0)
    else:
        qs, kr = [1], port.amplitude_damping(0.35)
    d = abi.DM(n)
    d.apply(ops)
    d.apply_channel(qs, kr)
    np.testing.assert_allclose(d.rho(), port.dm_apply_channel(rho0.copy(), qs, kr), atol=TOL, rtol=0)


def test_generic_two_qubit_channel_dense_path(port):
    # a non-depolarizing 2-qubit channel takes the dense 16x16 superoperator path
    n = 5
    ops = port.random_circuit(23, n, 30)
    rho0 = port.dm_run(n, ops)
    a = port.amplitude_damping(0.3)
    kr = np.array([np.kron(x, y) for x in a for y in a])
    d = abi.DM(n)
    d.apply(ops)
    d.apply_channel([4, 0], kr)
    np.testing.assert_allclose(d.rho(), port.dm_apply_channel(rho0.copy(), [4, 0], kr), atol=TOL, rtol=0)


def test_dm_reductions(port):
    n = 6
    ops = port.random_circuit(41, n, 40, 2)
    noise = NoiseSpec(n, e1=0.02, e2=0.04)
    want = port.dm_run_noisy(n, ops, noise)
    d = abi.DM(n)
    d.set_rho(want)
    assert abs(d.trace() - port.dm_trace(want)) < 1e-12
    assert abs(d.purity() - port.dm_purity(want)) < 1e-12
    assert abs(d.hermiticity_residual() - port.dm_hermiticity(want)) < 1e-15
    rng = np.random.default_rng(2)
    terms = [("".join(rng.choice(list("IXYZ"), size=n)), float(rng.uniform(-2, 2))) for _ in range(30)]
    re, im = d.expectations(terms)
    np.testing.assert_allclose(re, [port.dm_expectation(want, L, c) for L, c in terms], atol=TOL, rtol=0)
    assert np.max(np.abs(im)) < 1e-8
    np.testing.assert_allclose(d.probabilities(), port.dm_probabilities(want), atol=1e-14, rtol=0)


def test_readout_dist(port):
    n = 10
    rng = np.random.default_rng(4)
    p = rng.random(1 << n)
    p /= p.sum()
    p01 = rng.uniform(0, 0.1, n)
    p10 = rng.uniform(0, 0.1, n)
    p01[3] = p10[3] = 0.0
    np.testing.assert_allclose(abi.readout_apply_dist(p, p01, p10), port.readout_apply_dist(p, p01, p10),
                               atol=1e-15, rtol=0)
    with pytest.raises(abi.ContractError, match="sums to"):
        abi.readout_apply_dist(p * 1.1, p01, p10)


def test_dm_guard_and_errors():
    with pytest.raises(abi.ContractError):
        abi.DM(15)
    d = abi.DM(2)
    with pytest.raises(abi.ContractError, match="MEASURE"):
        d.apply([("measure", [0])])
    d.apply([("id", [0]), ("barrier", [0])])
    assert d.rho()[0, 0] == 1.0


@pytest.mark.parametrize("n,kind", [(6, "qaoa"), (8, "qaoa"), (7, "tfim"), (9, "tfim")])
def test_config_c4_circuits_noisy(port, n, kind):
    """BASELINE config C4 shapes (noisy TFIM Trotter / QAOA-MaxCut ring, device
    noise from a synthetic calibration) through the drop-in API, n >= 6 on the
    Hermitian (mirror) passes, against the oracle's blockwise Kraus sums."""
    from paper_2401_06861_b200 import naqs, workloads
    from oracle import list_to_ops

    ops = workloads.qaoa_ring(n, 2) if kind == "qaoa" else workloads.tfim_trotter(n, 0.3, steps=4)
    noise = NoiseSpec(n)
    circ = naqs.Circuit(n)
    for name, qs, ps in ops:
        circ.add(name, qs, ps)
    rho = naqs.run_density(circ, naqs.load_calibration(noise.calibration_json()))
    want = port.dm_run_noisy(n, list_to_ops(ops), noise)
    np.testing.assert_allclose(rho, want, atol=TOL, rtol=0)
