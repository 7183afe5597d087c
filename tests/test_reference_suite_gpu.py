"""The reference's own doctest suites (proj/tests/test_gates_pauli.cpp,
test_statevector.cpp, test_densitymatrix.cpp, test_noise.cpp, test_qasm.cpp,
test_bench.cpp, test_tfim.cpp, test_vqe.cpp, test_neldermead.cpp)
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


def test_bench_directory_over_the_corpus():
    """naqs.bench_directory (proj/src/bench.cpp semantics) on the QASM
    conformance corpus: accepted files are timed, rejected ones are skipped
    rows carrying the parser's diagnostic."""
    from paper_2401_06861_b200 import naqs

    corpus = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                          "qasm_tree", "tests", "data", "qasm")
    verdict = {}
    for line in open(os.path.join(corpus, "conformance.txt")):
        if line.strip() and not line.startswith("#"):
            parts = line.split(None, 2)
            verdict[parts[0][:-5]] = (parts[1], parts[2].strip() if len(parts) > 2 else "")
    rows = naqs.bench_directory(corpus, "sv", 2)
    assert [r["name"] for r in rows] == sorted(verdict)
    for r in rows:
        kind, reason = verdict[r["name"]]
        if kind == "accept":
            assert not r["skipped"] and len(r["times_ms"]) == 2 and r["median_ms"] >= r["min_ms"] >= 0
        else:
            assert r["skipped"] and reason in r["reason"]
    dm = naqs.bench_directory(corpus, "dm", 1)
    assert sum(not r["skipped"] for r in dm) == sum(v[0] == "accept" for v in verdict.values())
