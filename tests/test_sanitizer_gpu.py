"""compute-sanitizer over the CUDA paths at small n: memcheck
(out-of-bounds / misaligned device accesses, leaks of device allocations) and
racecheck (shared-memory hazards between the threads of a CTA -- the pass
kernels' relayouts) on a state-vector run through the generic and the
pass-specialised (NVRTC) kernels, the reductions, sampling, and a noisy
density-matrix run.  The child process uses only the C ABI (no torch)."""
import os
import shutil
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = textwrap.dedent(f"""
    import sys
    sys.path[:0] = [{ROOT!r}, {os.path.join(ROOT, 'oracle')!r}]
    import numpy as np
    from oracle import Port
    from paper_2401_06861_b200 import abi
    port = Port()
    for n, tile in [(12, 8), (13, 0)]:
        ops = port.random_circuit(5 + n, n, 120)
        sv = abi.SV(n, tile_qubits=tile)
        sv.apply(ops)
        got = sv.amplitudes()
        assert np.max(np.abs(got - port.sv_run(n, ops))) < 1e-10
        sv.expectations([("XYZ" + "I" * (n - 3), 0.5), ("Z" * n, 1.0)])
        sv.probabilities()
        sv.sample_sorted(np.sort(port.rng_double(3, 256)))
        sv.close()
    for n, tile in [(5, 0), (7, 6)]:
        ops = port.random_circuit(21, n, 40)
        dm = abi.DM(n, tile_qubits=tile)
        dm.apply(ops)
        dm.apply_channel([1], port.amplitude_damping(0.1))
        dm.trace(); dm.purity(); dm.probabilities()
        del dm
    print("CHILD_OK")
""")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_compute_sanitizer(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    args = [cs, "--tool", tool, "--error-exitcode", "3"]
    if tool == "memcheck":
        args += ["--leak-check", "full"]
    env = dict(os.environ, NQ_JIT="sync")  # specialised kernels compiled before their first launch
    r = subprocess.run(args + [sys.executable, "-c", CHILD], capture_output=True, text=True, timeout=1500, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "CHILD_OK" in out, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-4000:]
