"""Batches of small independent circuits (nq_batch_run)
against the oracle: state-vector expectations / probabilities and noisy
density-matrix probabilities / expectations, circuit by circuit, 1e-10."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import NoiseSpec, Port, Ref, ops_to_list  # noqa: E402

from paper_2401_06861_b200 import abi, naqs, workloads  # noqa: E402

pytestmark = pytest.mark.gpu


def test_sv_batch_matches_oracle():
    port = Port()
    n = 7
    circuits = [ops_to_list(port.random_circuit(300 + b, n, 40 + 3 * b)) for b in range(24)]
    terms = [("ZIIIIII", 1.0), ("XYZIIXI", 0.7), ("IIIYYII", -1.3)]
    out, _, pr = abi.batch_run(n, [[("gate", g) for g in c] for c in circuits], terms, probabilities=True)
    for b, c in enumerate(circuits):
        amps = port.sv_run(n, c)
        assert np.max(np.abs(pr[b] - np.abs(amps) ** 2)) <= 1e-12
        for j, (letters, co) in enumerate(terms):
            assert abs(out[b, j] - port.expectation(amps, letters, co)) <= 1e-10


def test_dm_batch_matches_oracle():
    port = Port()
    n = 4
    spec = NoiseSpec(n, e1=0.01, e2=0.05)
    circuits = [port.random_circuit(500 + b, n, 30, 2) for b in range(12)]
    model = naqs.load_calibration(spec.calibration_json())
    ncircs = []
    for c in circuits:
        cc = naqs.Circuit(n)
        for k, q, p in ops_to_list(c):
            cc.add(k, q, p)
        ncircs.append(cc)
    dists = naqs.batch_noisy_distributions(ncircs, model)
    for b, c in enumerate(circuits):
        rho = port.dm_run_noisy(n, c, spec)
        p = np.maximum(np.real(np.diag(rho.reshape(1 << n, 1 << n))), 0.0)
        p = p / p.sum()
        ref = port.readout_apply_dist(p, spec.p01, spec.p10)
        assert np.max(np.abs(dists[b] - ref)) <= 1e-10


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_tfim4_sweep_batched_matches_reference():
    cal = open(os.path.join(ROOT, "tests", "golden", "example_5q.json")).read()
    t_ref, ideal_ref, noisy_ref, _ = Ref().tfim_sweep(cal, 4)
    rows = np.array(workloads.tfim_sweep_rows_batched(naqs, 4, naqs.load_calibration(cal)))
    assert np.array_equal(rows[:, 0], t_ref)
    assert np.max(np.abs(rows[:, 1] - ideal_ref)) <= 1e-10
    assert np.max(np.abs(rows[:, 2] - noisy_ref)) <= 1e-10


def test_batch_contracts():
    with pytest.raises(abi.ContractError):
        abi.batch_run(13, [[("gate", ("h", [0], []))]], [("Z" + "I" * 12, 1.0)])
    with pytest.raises(abi.ContractError):
        abi.batch_run(7, [[("gate", ("h", [0], []))]], [("Z" + "I" * 6, 1.0)], dm=True)
    with pytest.raises(abi.ContractError):  # channels need dm
        abi.batch_run(2, [[("channel", [0], [np.eye(2)])]], [("ZI", 1.0)])
