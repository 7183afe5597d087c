"""Application layer above the boundary (csrc/apps.cpp), host parts on CPU.

naqs.minimize is our Nelder-Mead; oracle/_ref carries the reference's own
proj/src/neldermead.cpp.  On the same objective both must take exactly the
same steps: traces, best points and convergence flags are compared
bit for bit (restarts, shrinks, budget exhaustion, non-finite aborts).
"""
import math

import numpy as np
import pytest

from paper_2401_06861_b200 import naqs


def rosenbrock(x):
    return sum(100.0 * (x[i + 1] - x[i] ** 2) ** 2 + (1.0 - x[i]) ** 2 for i in range(len(x) - 1))


def plateau(x):
    # ties in the simplex ordering (stable sort keeps insertion order)
    return float(round(abs(x[0] - 0.3) * 4) + round(abs(x[1] + 0.7) * 4))


def sphere_shift(x):
    return sum((v - 0.1 * (i + 1)) ** 2 for i, v in enumerate(x))


def nan_after(k):
    calls = [0]

    def f(x):
        calls[0] += 1
        return math.nan if calls[0] == k else sphere_shift(x)

    return f


CASES = [
    (rosenbrock, [-1.2, 1.0], dict()),
    (rosenbrock, [0.0] * 5, dict(max_evals=700)),
    (plateau, [0.0, 0.0], dict(initial_step=0.5)),
    (sphere_shift, [0.5, -0.2, 0.3], dict(x_tol=1e-4, f_tol=1e-12)),
    (sphere_shift, [0.5, -0.2, 0.3, 1.0], dict(max_evals=23)),
    (lambda x: math.cos(3 * x[0]) + x[0] ** 2 * 0.1 + math.sin(x[1]) ** 2, [2.0, 1.0], dict(initial_step=2.0)),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_minimize_matches_reference_bit_for_bit(ref, case):
    f, x0, kw = CASES[case]
    mine = naqs.minimize(f, x0, **kw)
    trace, best, best_f, conv = ref.minimize(f, x0, **kw)
    assert np.array_equal(np.array(mine.trace), trace)
    assert mine.iterations == len(trace)
    assert np.array_equal(np.array(mine.best_params), best)
    assert mine.best_energy == best_f
    assert mine.converged == conv


def test_minimize_aborts_on_non_finite_like_reference(ref):
    mine = naqs.minimize(nan_after(9), [0.2, 0.4])
    trace, best, best_f, conv = ref.minimize(nan_after(9), [0.2, 0.4])
    assert len(mine.trace) == len(trace) == 9 and math.isnan(mine.trace[-1]) and math.isnan(trace[-1])
    assert np.array_equal(np.array(mine.trace[:-1]), trace[:-1])
    assert mine.diagnostic == "objective returned a non-finite value at evaluation 9"
    assert not mine.converged and not conv
    assert np.array_equal(np.array(mine.best_params), best) and mine.best_energy == best_f


def test_minimize_contract_errors():
    with pytest.raises(naqs.NaqsError, match="at least one dimension"):
        naqs.minimize(lambda x: 0.0, [])
    with pytest.raises(naqs.NaqsError, match="max_evals must be >= 1"):
        naqs.minimize(lambda x: 0.0, [1.0], max_evals=0)


def test_reference_python_surface_is_complete():
    # proj/python/naqs/__init__.py:7-51
    names = ["Circuit", "bench_directory", "DeviceNoiseModel", "GateKind", "MinimizeResult", "NaqsError",
             "density_expectation", "emit_qasm", "expectation", "load_calibration", "load_calibration_file",
             "minimize", "parse_qasm", "parse_qasm_file", "run_density", "run_statevector", "run_vqe", "sample",
             "tfim_ground_energy", "tfim_sweep"]
    assert [n for n in names if not hasattr(naqs, n)] == []
