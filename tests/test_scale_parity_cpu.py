"""Pins for the benchmark-scale parity checks (CPU only).

The QFT-30 check of tests/test_scale_parity_gpu.py and bench.py compares the
device state with a closed form (oracle.qft_closed_form) because the
reference engine needs minutes for the 2,220 ops at n = 30.  Here that closed
form is pinned to the reference build (oracle/_ref: proj/src compiled
unmodified) on the same circuit, full state, at small n.
"""
import importlib.util
import os

import numpy as np
import pytest

from oracle import list_to_ops, qft_closed_form

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _workloads():
    spec = importlib.util.spec_from_file_location(
        "nq_workloads", os.path.join(ROOT, "paper_2401_06861_b200", "workloads.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.mark.parametrize("n", [1, 2, 5, 8, 13])
def test_qft_closed_form_matches_port(port, n):
    ops = _workloads().qft(n)
    want = port.sv_run(n, list_to_ops(ops))
    got = qft_closed_form(n, np.arange(1 << n))
    assert np.max(np.abs(got - want)) <= 1e-13


@pytest.mark.parametrize("n", [6, 11, 16])
def test_qft_closed_form_matches_reference_build(ref, n):
    ops = _workloads().qft(n)
    want = ref.sv_run(n, list_to_ops(ops))
    got = qft_closed_form(n, np.arange(1 << n))
    assert np.max(np.abs(got - want)) <= 1e-13


def test_ref_handle_readers(ref):
    # the persistent-state readers used at benchmark scale agree with the
    # one-shot entry points
    n = 10
    ops = ref.random_circuit(2024, n, 60)
    full = ref.sv_run(n, ops)
    h = ref.sv_new(n)
    try:
        ref.sv_run_timed(h, ops)
        idx = np.array([0, 1, 5, 513, 1023])
        assert np.array_equal(ref.sv_gather(h, idx), full[idx])
        assert ref.sv_norm_sq_h(h) == pytest.approx(float(np.sum(np.abs(full) ** 2)), abs=1e-14)
        terms = [("Z" + "I" * (n - 1), 1.0), ("XY" + "I" * (n - 3) + "Z", 0.5)]
        assert np.array_equal(ref.sv_expectations_h(h, n, terms), ref.sv_expectations(n, ops, terms))
        ref.sv_reset_h(h)
        assert ref.sv_gather(h, [0])[0] == 1.0
    finally:
        ref.sv_free(h)
