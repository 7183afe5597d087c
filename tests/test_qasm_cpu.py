"""OpenQASM 2.0 frontend on the CPU: the reference's own
QASM test cases (proj/tests/test_qasm.cpp, compiled unmodified against our
headers into build/ref_tests_on_b200 with its conformance corpus as a
fixture), and the Python surface."""
import os
import subprocess

import pytest

from paper_2401_06861_b200 import naqs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "ref_tests_on_b200")
CORPUS = os.path.join(ROOT, "tests", "golden", "qasm_tree", "tests", "data", "qasm")

# every test case of test_qasm.cpp that does not simulate (the last one runs
# on the GPU in test_reference_suite_gpu.py)
CASES = ["canonical bell fragment", "angle expressions fold to constants", "unsupported statements carry",
         "parse failures all carry", "registers flatten in declaration order", "whole-register broadcast",
         "emit produces expected fragments", "parse(emit(c)) reproduces", "conformance corpus behaves",
         "mutated corpus files never crash"]


@pytest.mark.skipif(not os.path.exists(BIN), reason="reference test binary not built")
@pytest.mark.parametrize("case", CASES)
def test_reference_qasm_case(case):
    r = subprocess.run([BIN, f"--tc={case}"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 1 passed | 0 failed" in r.stdout, r.stdout


def test_corpus_through_python():
    accepted = rejected = 0
    for line in open(os.path.join(CORPUS, "conformance.txt")):
        if not line.strip() or line.startswith("#"):
            continue
        parts = line.split(None, 2)
        name, verdict = parts[0], parts[1]
        text = open(os.path.join(CORPUS, name)).read()
        if verdict == "accept":
            c = naqs.parse_qasm(text)
            assert naqs.parse_qasm(naqs.emit_qasm(c)).ops() == c.ops()
            accepted += 1
        else:
            with pytest.raises(naqs.QasmParseError) as e:
                naqs.parse_qasm(text)
            assert parts[2].strip() in str(e.value)
            assert str(e.value).startswith("line ")
            rejected += 1
    assert accepted >= 15 and rejected >= 5


def test_file_stem_names_the_circuit():
    c = naqs.parse_qasm_file(os.path.join(CORPUS, "ghz5.qasm"))
    assert c.name == "ghz5" and c.num_qubits == 5
