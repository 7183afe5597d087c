"""The reference's own doctest suites (proj/tests/test_gates_pauli.cpp,
test_statevector.cpp, test_densitymatrix.cpp, test_noise.cpp, test_qasm.cpp)
compiled unmodified against our headers and linked with our library
(paper_2401_06861_b200/csrc/Makefile target `droptests`): the drop-in proof
for the C++ boundary, run on the B200."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "ref_tests_on_b200")


@pytest.mark.skipif(not os.path.exists(BIN), reason="reference test binary not built")
def test_reference_suites_pass_on_b200():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-4000:], r.stderr[-4000:])
    assert " 0 failed" in r.stdout, r.stdout
