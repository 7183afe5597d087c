"""C1: the TFIM n=4 magnetization sweep (proj/src/tfim.cpp:139-184) with the
reference calibration example_5q.json, row by row against the reference
build (ideal and noisy columns within 1e-10)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Ref  # noqa: E402

from paper_2401_06861_b200 import naqs, workloads  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not Ref.available(), reason="oracle/_ref not built")
def test_tfim4_sweep_matches_reference():
    cal = open(os.path.join(ROOT, "tests", "golden", "example_5q.json")).read()
    t_ref, ideal_ref, noisy_ref, _ = Ref().tfim_sweep(cal, 4)
    rows = workloads.tfim_sweep_rows(naqs, 4, naqs.load_calibration(cal))
    assert len(rows) == len(t_ref) == 31
    got = np.array(rows)
    assert np.array_equal(got[:, 0], t_ref)
    assert np.max(np.abs(got[:, 1] - ideal_ref)) <= 1e-10
    assert np.max(np.abs(got[:, 2] - noisy_ref)) <= 1e-10
    assert abs(got[0, 2] - 0.959) <= 1e-12  # t = 0 noisy row (tests/test_tfim.cpp:143-158 shape)
