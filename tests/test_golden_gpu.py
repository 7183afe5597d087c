"""GPU results against the committed golden fixtures produced by the
reference engine itself (tests/golden/make_golden.py: the reference compiled
unmodified from its sources).  These run on the GPU box, where
/root/reference does not exist.

Tolerances: 1e-10 absolute on amplitudes, entries, expectations and
probabilities (north star); sampling counts exact.
"""
import json
import os

import numpy as np
import pytest

from oracle import NoiseSpec, ops_to_list
from paper_2401_06861_b200 import abi, naqs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-10


def load(name):
    return np.load(os.path.join(GOLD, name))


@pytest.mark.parametrize("name,n", [("ref_sv_n10_s2024_d200.npz", 10), ("ref_sv_n16_s4040_d300.npz", 16)])
def test_sv_fixture(name, n):
    g = load(name)
    sv = abi.SV(n)
    sv.apply(g["ops"])
    np.testing.assert_allclose(sv.amplitudes(), g["amps"], atol=TOL, rtol=0)
    terms = list(zip([str(x) for x in g["letters"]], g["coeff"]))
    np.testing.assert_allclose(sv.expectations(terms), g["expect"], atol=TOL, rtol=0)


@pytest.mark.parametrize("name,n", [("ref_sv_n10_s2024_d200.npz", 10), ("ref_sv_n16_s4040_d300.npz", 16)])
def test_sampling_fixture_through_python_surface(name, n):
    g = load(name)
    c = naqs.Circuit(n)
    for k, q, p in ops_to_list(g["ops"]):
        c.add(k, q, p)
    counts = naqs.sample(c, 20000, 7)
    dense = np.zeros(1 << n, dtype=np.uint64)
    for bits, cnt in counts.items():
        dense[int(bits, 2)] = cnt
    assert np.array_equal(dense, g["counts"])


@pytest.mark.parametrize("name,n", [("ref_dm_noisy_n4_s11.npz", 4), ("ref_dm_noisy_n6_s12.npz", 6)])
def test_dm_noisy_fixture_through_python_surface(name, n):
    g = load(name)
    c = naqs.Circuit(n)
    for k, q, p in ops_to_list(g["ops"]):
        c.add(k, q, p)
    model = naqs.load_calibration(NoiseSpec(n).calibration_json())
    rho = naqs.run_density(c, model)
    np.testing.assert_allclose(rho, g["rho"], atol=TOL, rtol=0)
    for L, coeff, want in zip([str(x) for x in g["letters"]], g["coeff"], g["expect"]):
        got = naqs.density_expectation(c, f"{float(coeff)!r}*{L}", model)
        assert abs(got - want) <= TOL


def test_dm_reductions_fixture():
    g = load("ref_dm_noisy_n6_s12.npz")
    d = abi.DM(6)
    d.set_rho(g["rho"])
    tr, pur, herm = g["scalars"]
    assert abs(d.trace() - tr) <= 1e-12
    assert abs(d.purity() - pur) <= 1e-12
    assert abs(d.hermiticity_residual() - herm) <= 1e-14
    np.testing.assert_allclose(d.probabilities(), g["probs"], atol=1e-14, rtol=0)


def test_readout_fixture():
    g = load("ref_readout_n8.npz")
    np.testing.assert_allclose(abi.readout_apply_dist(g["dist"], g["p01"], g["p10"]), g["out"], atol=1e-15, rtol=0)


def test_every_gate_independent_model_through_python_surface():
    # proj/tests/python/test_reference.py:127-131
    c = naqs.Circuit(3)
    for k, q, p in [("h", [0], []), ("x", [1], []), ("y", [2], []), ("z", [0], []), ("s", [1], []),
                    ("sdg", [2], []), ("t", [0], []), ("tdg", [1], []), ("id", [2], []), ("rx", [0], [0.3]),
                    ("ry", [1], [-0.7]), ("rz", [2], [1.1]), ("u1", [0], [0.4]), ("u2", [1], [0.2, -0.5]),
                    ("u3", [2], [1.2, 0.3, -0.8]), ("cx", [0, 1], []), ("cz", [1, 2], []), ("swap", [0, 2], []),
                    ("ccx", [0, 1, 2], []), ("cx", [2, 0], [])]:
        c.add(k, q, p)
    got = naqs.run_statevector(c)
    assert np.max(np.abs(got - np.load(os.path.join(GOLD, "every_gate_numpy_model.npy")))) < 1e-12


def test_python_smoke_semantics():
    # proj/tests/python/test_smoke.py: bell, deterministic sampling, depolarizing <Z>
    c = naqs.Circuit(2, "bell")
    c.add("h", [0]).add("cx", [0, 1])
    r = 2 ** -0.5
    assert np.allclose(naqs.run_statevector(c), [r, 0, 0, r])
    a = naqs.sample(c, 1000, 7)
    assert a == naqs.sample(c, 1000, 7) and sum(a.values()) == 1000 and set(a) <= {"00", "11"}
    model = naqs.load_calibration(json.dumps({
        "qubits": [{"t1_us": 1.0, "t2_us": 1.0, "readout_p01": 0.0, "readout_p10": 0.0}],
        "gates": [{"name": "x", "qubits": [0], "error": 0.15, "duration_ns": 0.0}]}))
    c1 = naqs.Circuit(1)
    c1.add("x", [0])
    assert naqs.density_expectation(c1, "Z", model) == pytest.approx(-(1 - 4 * 0.15 / 3), abs=1e-12)
