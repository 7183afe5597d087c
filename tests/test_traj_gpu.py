"""Batched Monte-Carlo trajectories (nq_traj_run) against
the oracle's sequential run_trajectory (proj/src/statevector.cpp:339-401) and
the density-matrix law (acceptance criterion 5,
tests/acceptance/acceptance_main.cpp:137-173)."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
from oracle import NoiseSpec, Port, list_to_ops  # noqa: E402

from paper_2401_06861_b200 import abi, naqs  # noqa: E402

pytestmark = pytest.mark.gpu


def noisy_schedule(port, gates, n, e1=0.02, e2=0.02, t1=60.0, t2=40.0, ns1=100.0, ns2=100.0):
    """attach_noise (noise.cpp:383-426): gate, depolarizing(error, arity), thermal per qubit."""
    items = []
    for g in gates:
        items.append(("gate", g))
        k = len(g[1])
        p, ns = (e1, ns1) if k == 1 else (e2, ns2)
        if k <= 2:  # (attach_noise rejects arity 3; the ccx here only gets thermal noise)
            items.append(("channel", list(g[1]), port.depolarizing(p, k)))
        for q in g[1]:
            items.append(("channel", [q], port.thermal_relaxation(t1, t2, ns)))
    return items


def sequential(port, n, items, ntraj, seed, letters):
    rng = port.rng_state(seed)
    amps_all, br_all, z = [], [], []
    for _ in range(ntraj):
        a = np.zeros(1 << n, dtype=np.complex128)
        a[0] = 1
        brs = []
        for it in items:
            if it[0] == "gate":
                port.sv_apply(a, list_to_ops([it[1]]))
            else:
                brs.append(port.kraus_trajectory(a, it[1], it[2], rng))
        amps_all.append(a)
        br_all.append(brs)
        z.append(port.expectation(a, letters))
    return np.array(amps_all), np.array(br_all), np.array(z)


def test_batch_matches_sequential_trajectories():
    port = Port()
    n = 5
    gates = [("h", [0], []), ("cx", [0, 1], []), ("rx", [2], [0.4]), ("cx", [1, 2], []), ("rz", [1], [0.9]),
             ("ccx", [0, 1, 3], []), ("u3", [4], [0.3, 0.2, 0.1]), ("swap", [3, 4], []), ("cz", [2, 4], []),
             ("ry", [3], [1.1]), ("y", [0], [])]
    items = noisy_schedule(port, gates, n, e1=0.05, e2=0.08)
    nch = sum(1 for it in items if it[0] == "channel")
    ntraj, seed = 64, 505
    u = port.rng_double(seed, ntraj * nch)
    terms = [("ZIIII", 1.0), ("XXIII", 0.5), ("IYZXI", -0.3)]
    out, br, am = abi.traj_run(n, items, ntraj, u, terms, branches=True, amplitudes=True)
    ref_amps, ref_br, ref_z = sequential(port, n, items, ntraj, seed, "ZIIII")
    assert np.array_equal(br, ref_br)  # same branch every channel, every trajectory
    assert np.max(np.abs(am - ref_amps)) <= 1e-10
    assert np.max(np.abs(out[:, 0] - ref_z)) <= 1e-10
    for j, (letters, c) in enumerate(terms):
        ref = np.array([port.expectation(a, letters, c) for a in ref_amps])
        assert np.max(np.abs(out[:, j] - ref)) <= 1e-10


def test_trajectory_average_matches_density_matrix():
    """Acceptance 5: the MC mean of <Z0> over 10^4 trajectories is within 3
    standard errors of the density-matrix value."""
    port = Port()
    n = 3
    gates = [("h", [0], []), ("cx", [0, 1], []), ("cx", [1, 2], []), ("rx", [0], [0.4]), ("rz", [1], [0.9]),
             ("cx", [0, 2], [])]
    items = noisy_schedule(port, gates, n)
    nch = sum(1 for it in items if it[0] == "channel")
    ntraj = 10000
    u = port.rng_double(505, ntraj * nch)
    out, _, _ = abi.traj_run(n, items, ntraj, u, [("ZII", 1.0)])
    z = out[:, 0]
    dm = abi.DM(n)
    dm.apply_schedule(items)
    re, _ = dm.expectations([("ZII", 1.0)])
    se = np.sqrt(max(z.var(), 0.0) / ntraj)
    assert abs(z.mean() - re[0]) <= 3 * se, (z.mean(), re[0], se)


def test_contract_errors():
    port = Port()
    with pytest.raises(abi.ContractError):
        abi.traj_run(14, [("gate", ("h", [0], []))], 1, np.zeros((1, 0)), [("Z" + "I" * 13, 1.0)])
    # a non-trace-preserving "channel" is rejected like the reference
    bad = [("gate", ("h", [0], [])), ("channel", [0], [0.5 * np.eye(2)])]
    with pytest.raises(abi.ContractError):
        abi.traj_run(2, bad, 2, np.full((2, 1), 0.3), [("ZI", 1.0)])
    del port


def test_python_api_acceptance5():
    """naqs.trajectory_expectations: acceptance criterion 5 through the drop-in
    Python surface (attach_noise + Rng(505) + 10^4 trajectories)."""
    import json

    n = 3
    cal = {"name": "acc5", "qubits": [{"t1_us": 60.0, "t2_us": 40.0, "readout_p01": 0.0, "readout_p10": 0.0}] * n,
           "default_1q": {"error": 0.02, "duration_ns": 100.0}, "default_2q": {"error": 0.02, "duration_ns": 100.0}}
    model = naqs.load_calibration(json.dumps(cal))
    c = naqs.Circuit(n)
    for name, qs, ps in [("h", [0], []), ("cx", [0, 1], []), ("cx", [1, 2], []), ("rx", [0], [0.4]),
                         ("rz", [1], [0.9]), ("cx", [0, 2], [])]:
        c.add(name, qs, ps)
    z = naqs.trajectory_expectations(c, ["ZII"], model, 10000, 505)[:, 0]
    dm = naqs.density_expectation(c, "ZII", model)
    se = np.sqrt(z.var() / len(z))
    assert abs(z.mean() - dm) <= 3 * se


@pytest.mark.skipif(not __import__("oracle").Ref.available(), reason="oracle/_ref not built")
def test_per_trajectory_parity_with_reference_build():
    """Row t equals trajectory t of the reference's own sequential loop
    (run_trajectory with one shared Rng), within 1e-10."""
    from oracle import Ref

    n = 4
    ops = [("h", [0], []), ("cx", [0, 1], []), ("ry", [2], [0.7]), ("cx", [1, 2], []), ("rz", [3], [0.2]),
           ("cx", [2, 3], []), ("u3", [1], [0.4, 0.1, -0.3]), ("swap", [0, 3], [])]
    spec = NoiseSpec(n, t1=50.0, t2=30.0, p01=0.0, p10=0.0, e1=0.03, d1=80.0, e2=0.05, d2=250.0)
    _, zref = Ref().traj_time(n, ops, spec, 2000, 777)
    c = naqs.Circuit(n)
    for name, qs, ps in ops:
        c.add(name, qs, ps)
    z = naqs.trajectory_expectations(c, ["Z" + "I" * (n - 1)], naqs.load_calibration(spec.calibration_json()),
                                     2000, 777)[:, 0]
    assert np.max(np.abs(z - zref)) <= 1e-10
